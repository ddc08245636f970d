set -x
cd $GRAFT_REPO_ROOT
timeout -k 5 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke26.log 2>&1 || { echo "SMOKE FAILED"; tail -30 gpurun_out/smoke26.log; exit 1; }
tail -1 gpurun_out/smoke26.log
timeout -k 5 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_abi.py -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest26.log 2>&1
echo "pytest rc=$?"; tail -15 gpurun_out/pytest26.log
for v in new r2 new r2; do
  if [ $v = new ]; then unset SALE_B200_LIB; else export SALE_B200_LIB=$PWD/paper_2505_24179_b200/lib_alt/libsale_b200_$v.so; fi
  timeout -k 5 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --sweep "" --no-e2e > gpurun_out/bench26_$v.json 2> gpurun_out/bench26_$v.err
  python -c "
import json; d=json.load(open('gpurun_out/bench26_$v.json')); s=d['stage_ms']; print('$v', round(d['value'],2), 'dense', round(d['dense_ms'],2), 'attn', round(s['attention'],2), 'est', round(s['estimate'],2), 'clk', d['clocks']['sm_mhz'], '64k', round(d['at_64k']['ms'],2), round(d['at_64k']['dense_ms'],2))"
done
unset SALE_B200_LIB
timeout -k 5 300 python profiles/attn_waits.py > gpurun_out/attn_waits26.txt 2>&1; cat gpurun_out/attn_waits26.txt
