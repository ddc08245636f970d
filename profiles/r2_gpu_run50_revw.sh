cd $GRAFT_REPO_ROOT
bash profiles/ab_run.sh revw new revw
for v in new revw; do
  if [ $v = new ]; then unset SALE_B200_LIB; else export SALE_B200_LIB=$PWD/paper_2505_24179_b200/lib_alt/libsale_b200_$v.so; fi
  timeout -k 5 600 ncu --clock-control none -k regex:sparse_attention -c 2 --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum python profiles/run_prefill.py --iters 1 --dense > gpurun_out/ncu50_$v.csv 2>/dev/null
  grep -E "dram__bytes_read|duration" gpurun_out/ncu50_$v.csv | awk -F'","' -v v=$v '{print v, $(NF-3), $(NF-2), $NF}'
done
