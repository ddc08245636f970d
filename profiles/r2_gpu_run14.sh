set -x
cd $GRAFT_REPO_ROOT
timeout -k 5 90 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke14.log 2>&1 || { echo "SMOKE FAILED"; exit 1; }
timeout -k 5 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c2.py -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest_gpu14.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu14.log
timeout -k 5 300 python profiles/est_waits.py 131072 > gpurun_out/est_waits14.txt 2>&1; cat gpurun_out/est_waits14.txt
timeout -k 5 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --sweep "" --no-e2e > gpurun_out/bench14.json 2> gpurun_out/bench14.err
python - <<'PY'
import json
d=json.load(open("gpurun_out/bench14.json"))
print(round(d["value"],2), "dense", round(d["dense_ms"],2), {k: round(v,2) for k,v in d["stage_ms"].items()}, "64k", d["at_64k"]["ms"], d["at_64k"]["stage_ms"])
PY
