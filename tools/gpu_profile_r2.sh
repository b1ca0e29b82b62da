# Round-2 ncu evidence (one GPU, never under a multi-rank command):
#  * launch list of the default bench command (C3)
#  * full captures: fused pair disjoint kernel (C3), singular generic kernels,
#    green_box_kernel (GCA)
#  * per-kernel DRAM bytes of h2 matvec (C3 SLP) and of the C4 P1 step
mkdir -p gpurun_out
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"
if [ "${LAUNCH:-1}" = "1" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu --no-matvec --no-separate > gpurun_out/launches_c3.log 2>&1
fi
if [ "${FULL:-1}" = "1" ]; then
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:disjoint_kernel -c 1 -o gpurun_out/prof_pair_c3 -f python tools/profile_step.py --config c3 > gpurun_out/ncu_pair_c3.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:generic_kernel -c 3 -o gpurun_out/prof_generic_c3 -f python tools/profile_step.py --config c3 > gpurun_out/ncu_generic_c3.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:green_box -c 2 -o gpurun_out/prof_green_c3 -f python tools/profile_step.py --config c3 > gpurun_out/ncu_green_c3.log 2>&1
fi
if [ "${AUX:-1}" = "1" ]; then
timeout 900 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/matvec_c3.csv python tools/matvec_step.py c3 > gpurun_out/matvec_c3.log 2>&1
timeout 900 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/p1_c4.csv python bench.py --config c4 --steps 1 --warmup 3 --e2e-steps 0 > gpurun_out/p1_c4.log 2>&1
fi
ls -la gpurun_out | head -40
