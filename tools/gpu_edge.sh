mkdir -p gpurun_out
for v in 0 1 0 1; do
  if [ $v = 1 ]; then export GCABEM_NO_GROUPED_EDGE=1; else unset GCABEM_NO_GROUPED_EDGE; fi
  timeout 600 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu --no-matvec --no-separate --no-secondary > gpurun_out/e.json 2> gpurun_out/e.err
  python -c "import json; d=json.load(open('gpurun_out/e.json')); print('no_grouped_edge=$v', round(d['ms_per_step'],3), round(d['roofline']['kernel_share_of_step'],3))"
done
