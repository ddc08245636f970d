set -x
cd $GRAFT_REPO_ROOT
timeout -k 5 90 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke10.log 2>&1 || { echo "SMOKE FAILED"; tail -20 gpurun_out/smoke10.log; exit 1; }
timeout -k 5 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu10.log 2>&1
echo "pytest rc=$?"
tail -8 gpurun_out/pytest_gpu10.log
# multi-GPU host logic on one GPU: 8 gloo ranks share the device (functional)
BENCH_DIST_BACKEND=gloo timeout -k 5 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 8 --steps 2 --warmup 1 --tokens 32768 --second-tokens 0 --no-cpu-baseline > gpurun_out/gloo8.json 2> gpurun_out/gloo8.err
echo "gloo8 rc=$?"; tail -c 1500 gpurun_out/gloo8.json
BENCH_DIST_BACKEND=gloo timeout -k 5 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 8 --model qwen --steps 2 --warmup 1 --tokens 32768 --second-tokens 0 --no-cpu-baseline > gpurun_out/gloo8_qwen.json 2> gpurun_out/gloo8_qwen.err
echo "gloo8 qwen rc=$?"; tail -c 1500 gpurun_out/gloo8_qwen.json
