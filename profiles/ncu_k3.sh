#!/bin/bash
# Key K3 metrics for one sparse + one dense launch of the bench workload (used per change).
ncu --clock-control none -k regex:sparse_attention -c 2 --csv \
  --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,lts__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum \
  python profiles/run_prefill.py --iters 1 --dense
