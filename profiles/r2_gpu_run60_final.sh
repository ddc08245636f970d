# round-2 final evidence: smoke, full GPU suite, the driver's bench command, tau sweeps,
# the reference arm, the ncu launch list and one ncu --set full capture
set -x
cd $GRAFT_REPO_ROOT
timeout -k 5 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke60.log 2>&1 || { echo "SMOKE FAILED"; tail -20 gpurun_out/smoke48.log; exit 1; }
tail -1 gpurun_out/smoke60.log
timeout -k 5 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu60.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu60.log
timeout -k 5 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2h_bench_main.json 2> gpurun_out/r2h_bench_main.err
echo "main rc=$?"
timeout -k 5 600 python bench.py --tokens 65536 --sweep 0.004,0.008,0.016,0.032,0.064 --second-tokens 0 --no-e2e --no-cpu-baseline > gpurun_out/r2h_c3_64k.json 2> gpurun_out/r2h_c3_64k.err
timeout -k 5 600 python bench.py --sweep 0.008,0.016,0.032,0.064 --second-tokens 0 --no-e2e --no-cpu-baseline > gpurun_out/r2h_c3_128k.json 2> gpurun_out/r2h_c3_128k.err
timeout -k 5 600 python bench.py --model qwen --sweep 0.004,0.016,0.032,0.064,0.128 --second-tokens 0 --no-e2e --no-cpu-baseline > gpurun_out/r2h_c4_qwen.json 2> gpurun_out/r2h_c4_qwen.err
timeout -k 5 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2h_ref_arm.json 2> gpurun_out/r2h_ref_arm.err
timeout -k 5 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2h_bench_launches.csv python bench.py --steps 2 --warmup 1 --sweep "" --second-tokens 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch60.log 2>&1
timeout -k 5 1500 ncu --set full --clock-control none --import-source on -c 6 -o gpurun_out/r2h_full python profiles/run_prefill.py --iters 1 --dense > gpurun_out/ncu_full60.log 2>&1
echo "ncu full rc=$?"
python profiles/ncu_summarize.py gpurun_out/r2h_full.ncu-rep gpurun_out/r2h_ncu_summary_table.md gpurun_out/ncu_traffic_r2h.json
cat gpurun_out/r2h_ncu_summary_table.md
echo done
