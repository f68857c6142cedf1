mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_integration.py -m gpu -q -x > gpurun_out/integ.log 2>&1; echo integ=$? > gpurun_out/status_integ.txt
tail -3 gpurun_out/integ.log >> gpurun_out/status_integ.txt
