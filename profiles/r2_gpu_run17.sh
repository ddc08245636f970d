set -x
cd $GRAFT_REPO_ROOT
timeout -k 5 90 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke17.log 2>&1 || { echo "SMOKE FAILED"; exit 1; }
timeout -k 5 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_abi.py tests/test_gpu_pipeline.py -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest_gpu17.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu17.log
for r in 1 2; do
timeout -k 5 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --sweep "0.064" --no-e2e > gpurun_out/bench17_$r.json 2> gpurun_out/bench17_$r.err
python -c "
import json; d=json.load(open('gpurun_out/bench17_$r.json')); print(round(d['value'],2), 'dense', round(d['dense_ms'],2), {k: round(v,2) for k,v in d['stage_ms'].items()}, d['tau_sweep'], d['at_64k']['stage_ms']['attention'])"
SALE_B200_LIB=$PWD/profiles/ab/r1src/paper_2505_24179_b200/lib/libsale_b200.so timeout -k 5 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --sweep "0.064" --no-e2e > gpurun_out/bench17_old_$r.json 2> gpurun_out/bench17_old_$r.err
python -c "
import json; d=json.load(open('gpurun_out/bench17_old_$r.json')); print('old', round(d['value'],2), 'dense', round(d['dense_ms'],2), {k: round(v,2) for k,v in d['stage_ms'].items()}, d['tau_sweep'], d['at_64k']['stage_ms']['attention'])"
done
