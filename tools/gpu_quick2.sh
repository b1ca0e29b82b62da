# quick e2e/value check of C3 and C2 (no cpu sample, no matvec)
mkdir -p gpurun_out
for cfg in c3 c2; do
timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --e2e-steps 3 --no-cpu --no-matvec > gpurun_out/q_$cfg.json 2> gpurun_out/q_$cfg.err
python -c "import json; d=json.load(open('gpurun_out/q_$cfg.json')); print('$cfg', round(d['ms_per_step'],3), '%.3e'%d['value'], round(d['roofline']['frac'],4), 'e2e %.3e'%d['e2e']['value'], d['e2e']['seconds_per_step'], d['e2e']['phases_s'], d['h2_setup']['total_s'], d['h2_setup']['total_warm_s'])" || tail -5 gpurun_out/q_$cfg.err
done
