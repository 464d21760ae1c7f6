# GPU round trip without profiling: parity tests + bench (+ tail probe).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} 2>&1 | tail -30 > gpurun_out/pytest_gpu.txt
cat gpurun_out/pytest_gpu.txt
timeout 600 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
if [ -n "$TAIL" ]; then timeout 600 python scripts/probe_tail.py > gpurun_out/tail.log 2>&1; cat gpurun_out/tail.log; fi
