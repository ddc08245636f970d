# longer sequences on one B200 (Llama layer, B = 1): 256K and 512K tokens
cd $GRAFT_REPO_ROOT
for n in 262144 524288; do
  timeout -k 5 1200 python bench.py --tokens $n --steps 3 --warmup 3 --sweep 0.004,0.064 --second-tokens 0 --no-cpu-baseline > gpurun_out/r2g_long_$n.json 2> gpurun_out/r2g_long_$n.err
  echo "n=$n rc=$?"; tail -2 gpurun_out/r2g_long_$n.err
done
