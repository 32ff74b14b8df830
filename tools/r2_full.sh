# round-2 evidence run (tests, bench, variant sweep); ncu captures go through tools/r2_ncu.sh
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_full.log 2>&1; echo rc=$? >> gpurun_out/gputest_full.log
timeout 300 python bench.py > gpurun_out/bench_r2.log 2>&1
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_r2.log 2>&1
GRAPH=1 timeout 900 python tools/bench_variants.py dense sweep cublas fused pair diag skinny tc gett > gpurun_out/variants_r2.log 2>&1
cp gpurun_out/variants.json gpurun_out/variants_r2.json
timeout 300 python tools/bench_variants.py simt host > gpurun_out/variants_simt_host.log 2>&1
timeout 300 python tools/host_overhead.py > gpurun_out/host_overhead.log 2>&1
