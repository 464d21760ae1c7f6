mkdir -p gpurun_out
timeout 900 python scripts/diag/c4_tail.py 4096 > gpurun_out/c4_tail.jsonl 2>&1; cat gpurun_out/c4_tail.jsonl | cut -c1-300
timeout 900 python -m pytest tests/test_gpu_nsga_large.py -x -q 2>&1 | tail -5
timeout 900 python bench.py --steps 2 --warmup 1 --cpu-seconds 10 > gpurun_out/bench_r2b.json 2> gpurun_out/bench_r2b.err; tail -5 gpurun_out/bench_r2b.err; cat gpurun_out/bench_r2b.json
