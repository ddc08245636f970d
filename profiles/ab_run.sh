#!/bin/bash
# A/B bench on one box: profiles/ab_run.sh <tag> <variant>... ; variant "new" = lib/, others lib_alt/libsale_b200_<v>.so
# optional env: PARITY=1 runs the GPU parity tests of the new build first; WAITS=1 the K3 cycle breakdown
cd $GRAFT_REPO_ROOT
tag=$1; shift
if [ -n "$PARITY" ]; then
  timeout -k 5 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1 || { echo "SMOKE FAILED"; tail -30 gpurun_out/smoke_$tag.log; exit 1; }
  tail -1 gpurun_out/smoke_$tag.log
  timeout -k 5 900 python -m pytest ${PARITY_TESTS:-tests/test_gpu_parity.py tests/test_gpu_abi.py} -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest_$tag.log 2>&1
  echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$tag.log
fi
for rep in 1 2; do
for v in "$@"; do
  if [ $v = new ]; then unset SALE_B200_LIB; else export SALE_B200_LIB=$PWD/paper_2505_24179_b200/lib_alt/libsale_b200_$v.so; fi
  timeout -k 5 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --sweep "" --no-e2e ${BENCH_ARGS} > gpurun_out/bench_${tag}_${v}_$rep.json 2> gpurun_out/bench_${tag}_${v}_$rep.err
  python -c "
import json; d=json.load(open('gpurun_out/bench_${tag}_${v}_$rep.json')); s=d['stage_ms']; print('$v', round(d['value'],2), 'dense', round(d['dense_ms'],2), {k: round(x,2) for k,x in s.items()}, 'clk', d['clocks']['sm_mhz'], '64k', round(d['at_64k']['ms'],2), round(d['at_64k']['dense_ms'],2), d['at_64k']['stage_ms'])"
done
done
unset SALE_B200_LIB
if [ -n "$WAITS" ]; then timeout -k 5 300 python profiles/attn_waits.py > gpurun_out/attn_waits_$tag.txt 2>&1; cat gpurun_out/attn_waits_$tag.txt; fi
