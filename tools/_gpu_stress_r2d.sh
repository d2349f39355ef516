mkdir -p gpurun_out
timeout 800 python tools/stress_forms.py 101 600 > gpurun_out/stress_forms_r2d.txt 2>&1
timeout 500 python tools/stress_api.py 102 300 > gpurun_out/stress_api_r2d.txt 2>&1
timeout 800 python tools/stress_codes.py 103 600 > gpurun_out/stress_codes_r2d.txt 2>&1
timeout 400 python tools/stress_tiles.py 104 200 > gpurun_out/stress_tiles_r2d.txt 2>&1
timeout 400 python tools/stress_misc.py 105 200 > gpurun_out/stress_misc_r2d.txt 2>&1
