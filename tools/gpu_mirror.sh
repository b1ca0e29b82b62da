# mirrored evaluation: GPU tests, then C3/C2 device step with and without it
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_mirror.py -q -x > gpurun_out/pytest_mirror.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_mirror.log
tail -15 gpurun_out/pytest_mirror.log
for cfg in c3 c2; do
  for m in "" "--no-mirror"; do
    timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --e2e-steps 2 --no-cpu --no-matvec --no-separate $m > gpurun_out/mir_${cfg}${m}.json 2> gpurun_out/mir_${cfg}${m}.err
    python -c "import json; d=json.load(open('gpurun_out/mir_${cfg}${m}.json')); print('$cfg $m', round(d['ms_per_step'],3), '%.3e'%d['value'], round(d['roofline']['frac'],4), round(d['roofline']['kernel_share_of_step'],3), 'e2e %.3e'%d['e2e']['value'])" || tail -5 gpurun_out/mir_${cfg}${m}.err
  done
done
if [ "${ALL:-0}" = "1" ]; then
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log; tail -5 gpurun_out/pytest_gpu.log
fi
