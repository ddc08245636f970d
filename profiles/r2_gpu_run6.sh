set -x
cd $GRAFT_REPO_ROOT
timeout 300 python profiles/attn_waits.py 131072 > gpurun_out/attn_waits6.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sparse_attention -c 2 -o gpurun_out/k3v2 python profiles/run_prefill.py --iters 1 --dense > gpurun_out/ncu_k3v2.log 2>&1
echo "ncu rc=$?"
