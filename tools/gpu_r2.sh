# Round-2 GPU pass: parity tests, default bench (C3), a 2-rank strong-scaling
# launch on one GPU (the torchrun path), the reference arm
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
if [ "${TESTS:-1}" = "1" ]; then
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
fi
timeout 900 python -X faulthandler bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
if [ "${STRONG:-1}" = "1" ]; then
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu --no-matvec --no-secondary > gpurun_out/bench_strong2.json 2> gpurun_out/bench_strong2.err; echo "strong2 rc=$?" >> gpurun_out/bench_strong2.err
fi
if [ "${REF:-1}" = "1" ]; then
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?" >> gpurun_out/bench_ref.err
fi
tail -3 gpurun_out/pytest_gpu.log; for f in bench bench_strong2 bench_ref; do echo "== $f"; cat gpurun_out/$f.json; tail -4 gpurun_out/$f.err; done
