# final evidence: default bench, reference arm, 2-rank launch on one GPU, ncu
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -X faulthandler bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?" >> gpurun_out/bench_ref.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu --no-matvec --no-secondary > gpurun_out/bench_strong2.json 2> gpurun_out/bench_strong2.err; echo "strong2 rc=$?" >> gpurun_out/bench_strong2.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu --no-matvec --no-separate --no-secondary > gpurun_out/launches_c3.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"disjoint_kernel|generic" -c 4 -o gpurun_out/prof_c3_final -f python tools/profile_step.py --config c3 > gpurun_out/ncu_final.log 2>&1
for f in bench bench_ref bench_strong2; do tail -c 600 gpurun_out/$f.json; echo; tail -1 gpurun_out/$f.err; done
