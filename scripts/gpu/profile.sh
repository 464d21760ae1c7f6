# Round-2 profile pass: issue counts of one bench step per workload (roofline
# input), the bench's launch list, one ncu --set full capture of the config-4
# interpreter launch (+ source lines), then the bench itself.
mkdir -p gpurun_out
M=smsp__inst_executed.sum,smsp__thread_inst_executed.sum,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for w in config4 config2; do
  timeout 900 ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file gpurun_out/issue_$w.csv python bench.py --profile-step $w > gpurun_out/issue_$w.log 2>&1
  python scripts/issue_profile.py $w gpurun_out/issue_$w.csv profiles/issue_per_launch.json > /dev/null && echo "issue profile $w ok"
done
cp profiles/issue_per_launch.json gpurun_out/issue_per_launch.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_ncu.log 2>&1; echo "launch list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:interp_tp --launch-skip 1 -c 1 -o gpurun_out/c4full -f python scripts/bench_configs.py config4 --steps 1 --cpu-seconds 0 > gpurun_out/c4full.log 2>&1; echo "ncu full rc=$?"
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err; cat gpurun_out/bench.json | cut -c1-600
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; cat gpurun_out/bench_ref.json | cut -c1-300
timeout 600 python scripts/diag/c4_sets.py > gpurun_out/c4_sets.jsonl 2> gpurun_out/c4_sets.err; echo "c4 sets rc=$?"
timeout 900 python scripts/bench_configs.py config3 --steps 3 > gpurun_out/config3.json 2> gpurun_out/config3.err; tail -1 gpurun_out/config3.json | cut -c1-300
timeout 900 python scripts/search_time.py --ref > gpurun_out/search_time.log 2>&1; echo "search rc=$?"
timeout 900 python scripts/nsga_bench.py > gpurun_out/nsga.jsonl 2> gpurun_out/nsga.err; echo "nsga rc=$?"
