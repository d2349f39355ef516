mkdir -p gpurun_out
timeout 1500 python tools/ber_codes.py r2c 1e8 > gpurun_out/ber_r2c.log 2>&1
cp profiles/r2c_ber_codes.json gpurun_out/ 2>/dev/null
timeout 900 python tools/ber_report.py r2c 1e9 > gpurun_out/ber_report_r2c.log 2>&1
cp profiles/r2c_ber*.json profiles/r2c_ber*.csv gpurun_out/ 2>/dev/null
