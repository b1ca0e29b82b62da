# GPU iteration: parity tests, then C2, C3 and C4 benches (no profiles)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python -X faulthandler bench.py --steps 5 --warmup 3 --cpu-seconds 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
if [ "${C3:-1}" = "1" ]; then
timeout 1200 python -X faulthandler bench.py --config c3 --steps 3 --warmup 3 --e2e-steps 3 --no-cpu > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "bench c3 rc=$?" >> gpurun_out/bench_c3.err
fi
if [ "${C4:-1}" = "1" ]; then
timeout 900 python -X faulthandler bench.py --config c4 --steps 5 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench c4 rc=$?" >> gpurun_out/bench_c4.err
fi
tail -5 gpurun_out/pytest_gpu.log; for f in bench bench_c3 bench_c4; do cat gpurun_out/$f.json; tail -3 gpurun_out/$f.err; done
