# A/B: the in-tree library vs a variant build (GCABEM_LIB_PATH), device step only
mkdir -p gpurun_out
VAR=${VAR:-abvar/libgcabem_b200.so}
for cfg in c2 c3; do
  for lib in base var; do
    if [ $lib = var ]; then export GCABEM_LIB_PATH=$PWD/$VAR; else unset GCABEM_LIB_PATH; fi
    timeout 900 python bench.py --config $cfg --steps 5 --warmup 3 --e2e-steps 0 --no-cpu --no-matvec > gpurun_out/ab_${cfg}_$lib.json 2> gpurun_out/ab_${cfg}_$lib.err
    python -c "import json; d=json.load(open('gpurun_out/ab_${cfg}_$lib.json')); print('$cfg $lib', round(d['ms_per_step'],3), round(d['roofline']['frac'],4))"
  done
done
