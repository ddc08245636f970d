cd $GRAFT_REPO_ROOT
timeout -k 5 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_abi.py tests/test_gpu_large.py -q -m gpu -p no:cacheprovider -x 2>&1 | tail -2
bash profiles/ab_run.sh rev new head
for v in new head; do
  if [ $v = new ]; then unset SALE_B200_LIB; else export SALE_B200_LIB=$PWD/paper_2505_24179_b200/lib_alt/libsale_b200_$v.so; fi
  timeout -k 5 600 ncu --clock-control none -k regex:sparse_attention -c 2 --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum python profiles/run_prefill.py --iters 1 --dense > gpurun_out/ncu49_$v.csv 2>/dev/null
  grep -E "dram__bytes|duration" gpurun_out/ncu49_$v.csv | awk -F'","' -v v=$v '{print v, $(NF-3), $(NF-2), $NF}'
done
