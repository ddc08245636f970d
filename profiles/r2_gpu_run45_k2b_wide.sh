cd $GRAFT_REPO_ROOT
timeout -k 5 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout -k 5 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_abi.py tests/test_gpu_pipeline.py -q -m gpu -p no:cacheprovider -x 2>&1 | tail -3
for rep in 1 2; do
for v in wide narrow; do
  if [ $v = narrow ]; then export SALE_B200_EST_NARROW=1; else unset SALE_B200_EST_NARROW; fi
  timeout -k 5 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --sweep "" --no-e2e > gpurun_out/bench45_${v}_$rep.json 2> gpurun_out/bench45_${v}_$rep.err
  python -c "
import json; d=json.load(open('gpurun_out/bench45_${v}_$rep.json')); s=d['stage_ms']; print('$v', round(d['value'],2), 'dense', round(d['dense_ms'],2), {k: round(x,2) for k,x in s.items()}, 'clk', d['clocks']['sm_mhz'], '64k', round(d['at_64k']['ms'],2), round(d['at_64k']['stage_ms']['estimate'],2), 'frac_est', round(d['estimator_roofline']['frac'],3))"
done; done
