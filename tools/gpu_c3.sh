# C3 (L7 Helmholtz kappa=4, orders 3/5) bench + Helmholtz kernel profile
mkdir -p gpurun_out
timeout 1500 python -X faulthandler bench.py --config c3 --steps 3 --warmup 3 --e2e-steps 2 --cpu-seconds 15 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "bench c3 rc=$?" >> gpurun_out/bench_c3.err
if [ "${PROFILE:-0}" = "1" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python tools/profile_step.py --config c3 > gpurun_out/launches_c3.log 2>&1
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:disjoint_kernel -c 2 -o gpurun_out/prof_disjoint_c3 -f python tools/profile_step.py --config c3 > gpurun_out/ncu_full_c3.log 2>&1
fi
cat gpurun_out/bench_c3.json; tail -5 gpurun_out/bench_c3.err
