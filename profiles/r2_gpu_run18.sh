set -x
cd $GRAFT_REPO_ROOT
timeout -k 5 90 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke18.log 2>&1 || { echo "SMOKE FAILED"; exit 1; }
tail -2 gpurun_out/smoke18.log
timeout -k 5 2000 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu18.log 2>&1
echo "pytest rc=$?"; grep -E "passed|failed|UserWarning: c" gpurun_out/pytest_gpu18.log | tail -8
timeout -k 5 900 python bench.py > gpurun_out/bench18.json 2> gpurun_out/bench18.err
echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench18.json')); print(round(d['value'],2), 'e2e', d['e2e']['value'], 'dense', round(d['dense_ms'],2), {k: round(v,2) for k,v in d['stage_ms'].items()}, d['roofline']['frac'], d['estimator_roofline']['frac'], d['clocks'])"
