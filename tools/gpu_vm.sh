mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_mirror.py tests/test_gpu_parity.py -q -x -k "mirror or L3 or pair_plan or c1" > gpurun_out/pytest_vm.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_vm.log; tail -15 gpurun_out/pytest_vm.log
timeout 900 python -m pytest tests/test_gpu_levels.py -q -x -k "c3 or c2" > gpurun_out/pytest_vm2.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_vm2.log; tail -3 gpurun_out/pytest_vm2.log
for cfg in c3 c2; do
  timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --e2e-steps 0 --no-cpu --no-matvec --no-separate > gpurun_out/g_$cfg.json 2> gpurun_out/g_$cfg.err
  python -c "import json; d=json.load(open('gpurun_out/g_$cfg.json')); print('$cfg', round(d['ms_per_step'],3), '%.3e'%d['value'], round(d['roofline']['frac'],4), round(d['roofline']['kernel_share_of_step'],3), d['flops_per_step'])" || tail -3 gpurun_out/g_$cfg.err
done
