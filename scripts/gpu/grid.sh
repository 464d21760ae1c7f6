mkdir -p gpurun_out
timeout 600 python scripts/diag/c4_tail.py 4096 2>&1 | grep -E "variants|active|late_cta" | cut -c1-400
timeout 3000 python scripts/config5_grid.py > gpurun_out/config5_grid.jsonl 2> gpurun_out/config5_grid.err; tail -3 gpurun_out/config5_grid.err; wc -l gpurun_out/config5_grid.jsonl
