mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_mirror.py tests/test_gpu_parity.py -q -x 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_levels.py -q -x -k "c3 or c2" 2>&1 | tail -2
for k in 1 2; do
timeout 600 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu --no-matvec --no-separate --no-secondary 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], '%.4e'%d['value'], d['roofline']['frac'], d['roofline']['kernel_share_of_step'], d['gpu_launches'])"
timeout 600 python bench.py --config c2 --steps 5 --warmup 3 --e2e-steps 0 --no-cpu --no-matvec --no-separate --no-secondary 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2', d['ms_per_step'], '%.4e'%d['value'], d['roofline']['frac'])"
done
