# ncu captures of the round-2 kernels, summarised on the box (the .ncu-rep files stay there)
mkdir -p /tmp/ncu
for c in dense8192 complex8192i dense1024; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 2 -c 1 -o /tmp/ncu/r2b_$c python tools/one_case.py $c > gpurun_out/ncu_$c.log 2>&1
  python tools/ncu_summary.py full /tmp/ncu/r2b_$c.ncu-rep gpurun_out/r2b_ncu_$c.json >> gpurun_out/ncu_$c.log 2>&1
done
ncu -i /tmp/ncu/r2b_dense8192.ncu-rep --page source --csv --print-source sass > /tmp/ncu/src.csv 2>/dev/null; gzip -c /tmp/ncu/src.csv > gpurun_out/r2b_dense8192_source.csv.gz
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches_bench.csv python bench.py --steps 5 --warmup 3 --e2e-steps 1 > gpurun_out/ncu_launches.log 2>&1
