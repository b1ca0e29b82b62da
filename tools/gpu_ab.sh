# A/B: the in-tree library vs variant builds under abvar/<name>/ (GCABEM_LIB_PATH),
# device step only, C3 by default (CFGS="c3 c2"), VARS="base x1 ..."
mkdir -p gpurun_out
for cfg in ${CFGS:-c3}; do
  for lib in ${VARS:-base}; do
    if [ $lib = base ]; then unset GCABEM_LIB_PATH; else export GCABEM_LIB_PATH=$PWD/abvar/$lib/libgcabem_b200.so; fi
    timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --e2e-steps 0 --no-cpu --no-matvec --no-separate --no-secondary > gpurun_out/ab_${cfg}_$lib.json 2> gpurun_out/ab_${cfg}_$lib.err
    python -c "import json; d=json.load(open('gpurun_out/ab_${cfg}_$lib.json')); print('$cfg $lib', round(d['ms_per_step'],3), round(d['roofline']['frac'],4), round(d['roofline']['kernel_share_of_step'],3))" || tail -3 gpurun_out/ab_${cfg}_$lib.err
  done
done
