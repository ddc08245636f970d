#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over every kernel at
# N in {1000, 2048}, Hq 8 / Hkv 2 (profiles/sanitize_run.py), with the
# sanitizer build of the library (longer mbarrier wait timeout). Logs go to
# gpurun_out/sanitize_<tool>_<N>.log; profiles/r2_sanitize_summary.txt is the
# committed summary.
set -u
cd "$(dirname "$0")/.."
make -s -C paper_2505_24179_b200 sanitize
export SALE_B200_LIB=$PWD/paper_2505_24179_b200/lib/libsale_b200_san.so
mkdir -p gpurun_out
for N in 1000 2048; do
  for tool in memcheck racecheck synccheck; do
    extra=""
    [ "$tool" = memcheck ] && extra="--leak-check full"
    # synccheck: K3's pv_done barrier is an event observed only when a rescale
    # or the epilogue needs it, which synccheck reports as a
    # "missing wait"; the other kernels are checked, K3 separately below
    [ "$tool" = synccheck ] && extra="--kernel-name-exclude kns=sparse_attention"
    timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool $tool $extra --target-processes all \
      --print-limit 50 python profiles/sanitize_run.py $N > gpurun_out/sanitize_${tool}_${N}.log 2>&1
    rc=$?
    echo "$tool N=$N rc=$rc :: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|LEAK SUMMARY|sanitize_run N|Error|error detected' gpurun_out/sanitize_${tool}_${N}.log | grep -v 'Host Frame' | sort | uniq -c | tr '\n' ' ')"
  done
done
