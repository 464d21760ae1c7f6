# Issue-count profile (bench roofline input), one full ncu capture of the
# dominant interpreter launch, then the bench with the fresh profile.
mkdir -p gpurun_out
timeout 600 ncu --metrics smsp__inst_executed.sum,smsp__thread_inst_executed.sum,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:interp --csv --log-file gpurun_out/issue.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/issue_bench.log 2>&1
python scripts/issue_profile.py gpurun_out/issue.csv gpurun_out/issue_per_launch.json && cp gpurun_out/issue_per_launch.json profiles/issue_per_launch.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:interp -s ${NCU_SKIP:-3} -c 1 -o gpurun_out/prof_interp python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; tail -2 gpurun_out/ncu_full.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
