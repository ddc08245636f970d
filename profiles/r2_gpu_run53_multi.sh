# multi-rank bench lines (gloo, ranks sharing the one GPU: functional, timings not meaningful),
# and config C5 (B=4 x 256K, all 32 units) on one B200
cd $GRAFT_REPO_ROOT
for n in 2 4 8; do
  BENCH_DIST_BACKEND=gloo timeout -k 5 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29520+n)) bench.py --gpus $n --steps 2 --warmup 1 --tokens 32768 --second-tokens 0 --no-cpu-baseline > gpurun_out/r2g_gloo${n}_llama.json 2> gpurun_out/r2g_gloo${n}_llama.err
  echo "gloo$n rc=$?"
done
BENCH_DIST_BACKEND=gloo timeout -k 5 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29530 bench.py --gpus 8 --model qwen --steps 2 --warmup 1 --tokens 32768 --second-tokens 0 --no-cpu-baseline > gpurun_out/r2g_gloo8_qwen.json 2> gpurun_out/r2g_gloo8_qwen.err
echo "gloo8 qwen rc=$?"
timeout -k 5 1200 python bench.py --batch 4 --tokens 262144 --steps 3 --warmup 1 --sweep "" --second-tokens 0 --no-cpu-baseline > gpurun_out/r2g_c5_b4_256k_1gpu.json 2> gpurun_out/r2g_c5.err
echo "c5 rc=$?"
