set -x
cd $GRAFT_REPO_ROOT
nvidia-smi > gpurun_out/smi.txt
nproc > gpurun_out/nproc.txt
nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_event_reasons.sw_power_cap --format=csv,noheader -lms 200 > gpurun_out/i8_clocks.csv &
SMI=$!
timeout 120 ./profiles/i8_peak > gpurun_out/i8_peak.json 2> gpurun_out/i8_peak.err
kill $SMI
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?"
timeout 2400 bash profiles/sanitize.sh > gpurun_out/sanitize_summary.txt 2>&1
echo "sanitize rc=$?"
