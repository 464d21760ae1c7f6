# Round-2 first GPU pass: parity suite (incl. the wide-thread conflict cases),
# smoke, config-4 throughput at BASELINE shape and one ncu --set full capture
# of a config-4 interpreter launch (reduced pop so the replay stays short).
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_wide_conflicts.py -x -q 2>&1 | tail -15 > gpurun_out/pytest_wide.txt; cat gpurun_out/pytest_wide.txt
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.txt; cat gpurun_out/pytest_gpu.txt
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 600 python scripts/bench_configs.py config4 --steps 2 --cpu-seconds 0 > gpurun_out/c4.json 2> gpurun_out/c4.err; tail -3 gpurun_out/c4.err; cat gpurun_out/c4.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:interp_tp -c 1 -o gpurun_out/c4full -f python scripts/bench_configs.py config4 --pop 592 --steps 1 --cpu-seconds 0 > gpurun_out/c4ncu.log 2>&1; tail -3 gpurun_out/c4ncu.log
