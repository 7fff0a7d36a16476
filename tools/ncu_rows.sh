#!/bin/bash
# Key ncu counters of every row kernel (one launch each, after the counting
# launch), for profiles/<TAG>_rows_ncu.txt (tools/ncu_rows_summary.py).
set -u
TAG=${1:-r2}
M=gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__thread_inst_executed_per_inst_executed.ratio,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,launch__registers_per_thread,launch__occupancy_limit_registers,launch__occupancy_limit_shared_mem,smsp__inst_executed.sum,launch__shared_mem_per_block_dynamic
for cfg in c4_tau c4_tau_bin c4_ode c1_tau128 c1_ssa128 c2 c3_lsoda c3s_lsoda c3s_ode c3_ode c1_hybrid256 c1_cle c5_tau c5_ode; do
  timeout 600 ncu --metrics $M --clock-control none -k "regex:kin_jit_stoch|kin_jit_hybrid|kin_jit_lsoda|stochastic_kernel|dopri5_kernel|lsoda_kernel|hybrid_kernel|cle_kernel" \
      --launch-skip 1 --launch-count 1 --csv python tools/quick_time.py $cfg > gpurun_out/${TAG}_ncu_$cfg.csv 2> gpurun_out/${TAG}_ncu_$cfg.err
  echo "$cfg rc=$?"
done
