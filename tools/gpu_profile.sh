# ncu evidence for profiles/: launch lists of the bench command itself (C2, C3)
# and full captures of the disjoint kernels: the fused pair plan the bench
# times (1 launch) and the separate single-layer plans (2 launches)
mkdir -p gpurun_out
for cfg in c2 c3; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$cfg.csv python bench.py --config $cfg --steps 1 --warmup 3 --e2e-steps 0 --no-cpu --no-matvec > gpurun_out/launches_$cfg.log 2>&1
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:disjoint_kernel -c 1 -o gpurun_out/prof_pair_$cfg -f python tools/profile_step.py --config $cfg > gpurun_out/ncu_pair_$cfg.log 2>&1
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:disjoint_kernel -c 2 -o gpurun_out/prof_disjoint_$cfg -f python tools/profile_step.py --config $cfg --separate > gpurun_out/ncu_full_$cfg.log 2>&1
done
ls -la gpurun_out
