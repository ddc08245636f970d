set -x
cd $GRAFT_REPO_ROOT
for v in base s3 s5 base s3 s5; do
  if [ $v = base ]; then unset SALE_B200_LIB; else export SALE_B200_LIB=$PWD/paper_2505_24179_b200/lib_alt/libsale_b200_$v.so; fi
  timeout -k 5 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --sweep "" --no-e2e > gpurun_out/bench24_$v.json 2> gpurun_out/bench24_$v.err
  python -c "
import json; d=json.load(open('gpurun_out/bench24_$v.json')); s=d['stage_ms']; print('$v', round(d['value'],2), 'dense', round(d['dense_ms'],2), 'stats', round(s['stats'],2), 'est', round(s['estimate'],2), 'attn', round(s['attention'],2), '64k stats', round(d['at_64k']['stage_ms']['stats'],2))"
done
