mkdir -p gpurun_out
for m in "" "--no-mirror" "" "--no-mirror"; do
timeout 600 python bench.py --steps 3 --warmup 3 --e2e-steps 5 --no-cpu --no-matvec --no-separate --no-secondary $m > gpurun_out/e2e.json 2> gpurun_out/e2e.err
python -c "import json; d=json.load(open('gpurun_out/e2e.json')); print('mirror' if '$m'=='' else 'plain', d['e2e']['seconds_per_step'], d['e2e']['phases_s'])"
grep "e2e step" gpurun_out/e2e.err | sed 's/\[{.*//'
done
