set -x
cd $GRAFT_REPO_ROOT
timeout -k 5 90 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke22.log 2>&1 || { echo "SMOKE FAILED"; exit 1; }
tail -1 gpurun_out/smoke22.log
timeout -k 5 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu22.log 2>&1
echo "pytest rc=$?"; grep -E "passed|failed|UserWarning: c" gpurun_out/pytest_gpu22.log | tail -6
timeout -k 5 900 python bench.py > gpurun_out/bench22.json 2> gpurun_out/bench22.err
python -c "
import json; d=json.load(open('gpurun_out/bench22.json')); print(round(d['value'],2), 'e2e', round(d['e2e']['value'],2), 'dense', round(d['dense_ms'],2), {k: round(v,2) for k,v in d['stage_ms'].items()}, round(d['roofline']['frac'],3), round(d['estimator_roofline']['frac'],3), d['clocks'], d['at_64k']['ms'], d['tau_sweep'])"
