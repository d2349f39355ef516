mkdir -p gpurun_out
timeout 900 python tools/stress_forms.py 21 480 > gpurun_out/stress_forms_r2b.txt 2>&1
timeout 600 python tools/stress_api.py 5 240 > gpurun_out/stress_api_r2b.txt 2>&1
