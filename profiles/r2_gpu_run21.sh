set -x
cd $GRAFT_REPO_ROOT
for v in p4 p6 p7 p8 p9 p4 p6 p7 p8 p9; do
  if [ $v = base ]; then unset SALE_B200_LIB; else export SALE_B200_LIB=$PWD/paper_2505_24179_b200/lib_alt/libsale_b200_$v.so; fi
  timeout -k 5 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --sweep "0.064" --no-e2e > gpurun_out/bench21_$v.json 2> gpurun_out/bench21_$v.err
  python -c "
import json; d=json.load(open('gpurun_out/bench21_$v.json')); print('$v', round(d['value'],2), 'dense', round(d['dense_ms'],2), 'attn', round(d['stage_ms']['attention'],2), 't064', round(d['tau_sweep'][0]['ms'],2), '64k', round(d['at_64k']['stage_ms']['attention'],2), round(d['at_64k']['dense_ms'],2))"
done
