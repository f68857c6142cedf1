timeout 400 python -m pytest tests/test_gpu_parity.py -q -x -k "keyswitch" > gpurun_out/kstc_tests.log 2>&1
echo "tests rc=$?" ; tail -2 gpurun_out/kstc_tests.log
timeout 300 python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-locpir > gpurun_out/kb_c.log 2>&1
python -c "
import json;d=json.loads(open('gpurun_out/kb_c.log').read().strip().splitlines()[-1]);k=d['keyswitch'];print('value',round(d['value']),'ks_ms',round(k['avg_launch_ms'],3),'tensor_frac',round(k['tensor_view']['frac'],3),'correct',d['correct'])"
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct \
    --clock-control none -k regex:"^k_keyswitch_tc$" --launch-skip 1 -c 2 --csv --log-file gpurun_out/kt_c.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-locpir > gpurun_out/kt_c.log 2>&1; echo traffic=$?
bash tools/selfcheck.sh > /dev/null 2>&1; tail -2 gpurun_out/selfcheck.txt
