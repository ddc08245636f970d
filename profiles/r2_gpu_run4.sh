set -x
cd $GRAFT_REPO_ROOT
timeout 300 python profiles/est_waits.py 131072 > gpurun_out/est_waits4.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shim.py tests/test_gpu_c2.py -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest_gpu4.log 2>&1
echo "pytest rc=$?"
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --sweep "" > gpurun_out/bench4.json 2> gpurun_out/bench4.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sink_local_stats -c 1 -o gpurun_out/k2a_r2b python profiles/run_prefill.py --iters 1 > gpurun_out/ncu_k2a.log 2>&1
timeout 2400 bash profiles/sanitize.sh > gpurun_out/sanitize_summary4.txt 2>&1
