# e2e (chunked host pipeline) with other chunk schedules at 128K
cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for v in new chk1 chk2; do
  if [ $v = new ]; then unset SALE_B200_LIB; else export SALE_B200_LIB=$PWD/paper_2505_24179_b200/lib_alt/libsale_b200_$v.so; fi
  timeout -k 5 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --sweep "" --second-tokens 0 > gpurun_out/bench58_${v}_$rep.json 2> gpurun_out/bench58_${v}_$rep.err
  python -c "
import json; d=json.load(open('gpurun_out/bench58_${v}_$rep.json')); print('$v', round(d['value'],2), 'e2e', round(d['e2e']['value'],2), 'clk', d['clocks']['sm_mhz'])"
done; done
