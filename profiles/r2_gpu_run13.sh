set -x
cd $GRAFT_REPO_ROOT
timeout -k 5 90 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke13.log 2>&1 || { echo "SMOKE FAILED"; exit 1; }
timeout -k 5 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2_bench_main.json 2> gpurun_out/r2_bench_main.err
echo "main rc=$?"
timeout -k 5 600 python bench.py --tokens 65536 --sweep 0.004,0.008,0.016,0.032,0.064 --second-tokens 0 --no-e2e --no-cpu-baseline > gpurun_out/r2_c3_64k.json 2> gpurun_out/r2_c3_64k.err
timeout -k 5 600 python bench.py --sweep 0.008,0.016,0.032,0.064 --second-tokens 0 --no-e2e --no-cpu-baseline > gpurun_out/r2_c3_128k.json 2> gpurun_out/r2_c3_128k.err
timeout -k 5 600 python bench.py --model qwen --sweep 0.004,0.016,0.032,0.064,0.128 --second-tokens 0 --no-e2e --no-cpu-baseline > gpurun_out/r2_c4_qwen.json 2> gpurun_out/r2_c4_qwen.err
timeout -k 5 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2_ref_arm.json 2> gpurun_out/r2_ref_arm.err
echo done
