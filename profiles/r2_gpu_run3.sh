set -x
cd $GRAFT_REPO_ROOT
timeout 300 python profiles/est_waits.py 131072 > gpurun_out/est_waits3.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shim.py -q -m gpu -p no:cacheprovider -k "geometry or shim or selection" > gpurun_out/pytest_gpu3.log 2>&1
echo "pytest rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sink_local_stats -c 1 -o gpurun_out/k2a_r2 python profiles/run_prefill.py --iters 1 > gpurun_out/ncu_k2a.log 2>&1
echo "ncu rc=$?"
export SALE_B200_LIB=$PWD/paper_2505_24179_b200/lib/libsale_b200_san.so
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool synccheck python profiles/sanitize_run.py 1000 > gpurun_out/sanitize_synccheck_1000.log 2>&1
echo "synccheck rc=$?"; tail -3 gpurun_out/sanitize_synccheck_1000.log
