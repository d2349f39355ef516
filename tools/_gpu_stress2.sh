mkdir -p gpurun_out
timeout 900 python tools/stress_forms.py 33 600 > gpurun_out/stress_forms_r2c.txt 2>&1
timeout 600 python tools/stress_misc.py 7 200 > gpurun_out/stress_misc_r2c.txt 2>&1
