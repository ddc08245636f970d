set -x
cd $GRAFT_REPO_ROOT
for v in base p0 p2 p3 base; do
  if [ $v = base ]; then unset SALE_B200_LIB; else export SALE_B200_LIB=$PWD/paper_2505_24179_b200/lib_alt/libsale_b200_$v.so; fi
  timeout -k 5 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --sweep "" --second-tokens 0 --no-e2e > gpurun_out/bench19_$v.json 2> gpurun_out/bench19_$v.err
  python -c "
import json; d=json.load(open('gpurun_out/bench19_$v.json')); print('$v', round(d['value'],2), 'dense', round(d['dense_ms'],2), 'attn', round(d['stage_ms']['attention'],2))"
done
