mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_mirror.py tests/test_gpu_parity.py tests/test_gpu_levels.py -q -x -k "not c5 and not pivots" > gpurun_out/ph.log 2>&1; echo "rc=$?" >> gpurun_out/ph.log; tail -3 gpurun_out/ph.log
for v in 0 1 0; do
  if [ $v = 1 ]; then export GCABEM_NO_SYM_HALF=1; else unset GCABEM_NO_SYM_HALF; fi
  timeout 600 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu --no-matvec --no-separate --no-secondary > gpurun_out/e.json 2> gpurun_out/e.err
  python -c "import json; d=json.load(open('gpurun_out/e.json')); print('no_half=$v', round(d['ms_per_step'],3), '%.4e'%d['value'], round(d['roofline']['kernel_share_of_step'],3), d['flops_per_step'])"
done
