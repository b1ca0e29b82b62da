# C5: L8 sphere (524,288 triangles), Helmholtz kappa=4 SLP+DLP, order sweep
# (disjoint n = singular n); device value + H2 setup (e2e skipped: 2 x 15 GB host payloads)
mkdir -p gpurun_out
for n in ${ORDERS:-3 4 5 6 7}; do
  timeout 1500 python -X faulthandler bench.py --config c5 --order $n --steps 2 --warmup 3 --e2e-steps 0 --no-cpu --no-matvec --no-separate --no-secondary ${EXTRA:-} > gpurun_out/bench_c5_n$n.json 2> gpurun_out/bench_c5_n$n.err
  echo "c5 n=$n rc=$?"; cat gpurun_out/bench_c5_n$n.json; tail -2 gpurun_out/bench_c5_n$n.err
done
