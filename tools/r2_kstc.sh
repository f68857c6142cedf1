# K2t bring-up: the key-switch parity tests, then an A/B of the bench with K2t on / off
timeout 400 python -m pytest tests/test_gpu_parity.py -q -x -k "keyswitch" > gpurun_out/kstc_tests.log 2>&1
echo "tests rc=$?" ; tail -5 gpurun_out/kstc_tests.log
bash tools/ab_env.sh LOCPIR_B200_KSTC 1 0
cat gpurun_out/ab.txt
