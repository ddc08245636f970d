set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_abi.py -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest_gpu5.log 2>&1
echo "pytest rc=$?"
tail -30 gpurun_out/pytest_gpu5.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --sweep "0.064" --no-e2e > gpurun_out/bench5_new.json 2> gpurun_out/bench5_new.err
SALE_B200_LIB=$PWD/profiles/ab/r1src/paper_2505_24179_b200/lib/libsale_b200.so timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --sweep "0.064" --no-e2e > gpurun_out/bench5_old.json 2> gpurun_out/bench5_old.err
python - <<'PY'
import json
for n in ("new","old"):
    try:
        d=json.load(open(f"gpurun_out/bench5_{n}.json"))
        print(n, round(d["value"],2), "dense", round(d["dense_ms"],2), {k: round(v,2) for k,v in d["stage_ms"].items()}, "sweep", d["tau_sweep"], "64k", d["at_64k"]["ms"], d["at_64k"]["dense_ms"])
    except Exception as e: print(n, "failed", e)
PY
