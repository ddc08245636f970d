set -x
cd $GRAFT_REPO_ROOT
make -s -C paper_2505_24179_b200 -j16 2>&1 | grep -E "error" 
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_abi.py tests/test_gpu_c2.py -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu2.log 2>&1
echo "pytest rc=$?"
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --sweep "" > gpurun_out/bench2.json 2> gpurun_out/bench2.err
echo "bench rc=$?"
timeout 2400 bash profiles/sanitize.sh > gpurun_out/sanitize_summary.txt 2>&1
echo "sanitize rc=$?"
