set -x
cd $GRAFT_REPO_ROOT
timeout -k 5 90 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke15.log 2>&1 || { echo "SMOKE FAILED"; exit 1; }
timeout -k 5 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_abi.py -q -m gpu -p no:cacheprovider -x -k "host or chunk or stale or geometry" > gpurun_out/pytest_gpu15.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu15.log
timeout -k 5 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --sweep "" > gpurun_out/bench15.json 2> gpurun_out/bench15.err
python - <<'PY'
import json
d=json.load(open("gpurun_out/bench15.json"))
print(round(d["value"],2), "e2e", round(d["e2e"]["value"],2), "dense", round(d["dense_ms"],2), {k: round(v,2) for k,v in d["stage_ms"].items()})
PY
