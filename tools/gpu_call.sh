mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_metric_range.py tests/test_fileio.py -m gpu -q -x > gpurun_out/pytest.log 2>&1; echo "rc $?" >> gpurun_out/pytest.log
timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-other-configs > gpurun_out/b.json 2>&1
ncu --metrics gpu__time_duration.sum,sm__inst_executed.avg.per_cycle_active,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio,smsp__inst_executed.sum --clock-control none -k regex:vtk16 -s 3 -c 1 --csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-other-configs > gpurun_out/ncu_q.csv 2>&1
