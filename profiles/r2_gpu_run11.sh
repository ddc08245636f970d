set -x
cd $GRAFT_REPO_ROOT
timeout -k 5 300 python profiles/est_waits.py 131072 > gpurun_out/est_waits11.txt 2>&1
timeout -k 5 300 python profiles/attn_waits.py 131072 > gpurun_out/attn_waits11.txt 2>&1
timeout -k 5 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_bench_launches.csv python bench.py --steps 2 --warmup 1 --sweep "" --second-tokens 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?"
timeout -k 5 1500 ncu --set full --clock-control none --import-source on -c 6 -o gpurun_out/r2_full python profiles/run_prefill.py --iters 1 --dense > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?"
python profiles/ncu_summarize.py gpurun_out/r2_full.ncu-rep gpurun_out/r2_ncu_summary_table.md gpurun_out/ncu_traffic_r2.json
cat gpurun_out/r2_ncu_summary_table.md
