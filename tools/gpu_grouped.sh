mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_mirror.py -q -x -k "L3 or pair_plan or mirrored or golden or raw" > gpurun_out/pytest_grp.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_grp.log; tail -3 gpurun_out/pytest_grp.log
for v in 0 1 0; do
  if [ $v = 1 ]; then export GCABEM_NO_GROUPED=1; else unset GCABEM_NO_GROUPED; fi
  for cfg in c3 c2; do
  timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --e2e-steps 0 --no-cpu --no-matvec --no-separate > gpurun_out/g_$cfg.json 2> gpurun_out/g_$cfg.err
  python -c "import json; d=json.load(open('gpurun_out/g_$cfg.json')); print('$cfg nogrouped=$v', round(d['ms_per_step'],3), '%.3e'%d['value'], round(d['roofline']['frac'],4), round(d['roofline']['kernel_share_of_step'],3))" || tail -3 gpurun_out/g_$cfg.err
  done
done
