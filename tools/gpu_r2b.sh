# default bench (C3) + C2 + reference arm + ncu of the mirrored pair kernel
mkdir -p gpurun_out
timeout 900 python -X faulthandler bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 900 python -X faulthandler bench.py --config c2 --steps 5 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "bench rc=$?" >> gpurun_out/bench_c2.err
if [ "${REF:-0}" = "1" ]; then
timeout 900 python bench.py --impl reference --config c2 --steps 3 --warmup 1 > gpurun_out/bench_ref_c2.json 2> gpurun_out/bench_ref_c2.err
fi
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu --no-matvec --no-separate > gpurun_out/launches_c3.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:disjoint_kernel -c 2 -o gpurun_out/prof_pair_c3_mir -f python tools/profile_step.py --config c3 > gpurun_out/ncu_pair_c3.log 2>&1
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/traffic_c2.csv -k regex:disjoint_kernel python tools/profile_step.py --config c2 > gpurun_out/traffic_c2.log 2>&1
for f in bench bench_c2; do cat gpurun_out/$f.json; tail -2 gpurun_out/$f.err; done
