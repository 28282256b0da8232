#!/bin/bash
# Summary of one ncu --set full report: durations, issue, stall reasons, DRAM bytes, SMEM wavefronts.
# usage: tools/ncu_summary.sh REPORT.ncu-rep
f=$1
ncu -i $f --page details --csv 2>/dev/null | grep -E '"(Duration|Executed Ipc Active|Issue Slots Busy|DRAM Throughput|No Eligible|Active Warps Per Scheduler|Eligible Warps Per Scheduler|Executed Instructions|Registers Per Thread|Dynamic Shared Memory Per Block)"' | awk -F'","' '{print $(NF-2)" | "$(NF-1)" | "$NF}'
ncu -i $f --page raw --csv 2>/dev/null | python3 -c "
import csv,sys
r=list(csv.reader(sys.stdin))
h=r[0]; v=r[2]
d=dict(zip(h,v))
st={k:float(d[k]) for k in h if k.startswith('smsp__average_warps_issue_stalled_') and k.endswith('_per_issue_active.ratio')}
for k,val in sorted(st.items(), key=lambda x:-x[1])[:8]: print(k.replace('smsp__average_warps_issue_stalled_','stall ').replace('_per_issue_active.ratio',''), round(val,3))
for k in ['dram__bytes_read.sum','smsp__inst_executed.sum','l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum','l1tex__data_pipe_lsu_wavefronts_mem_shared.sum','sm__pipe_tensor_op_hmma_cycles_active.avg.pct','sm__inst_executed_pipe_alu.avg.pct','sm__pipe_alu_cycles_active.avg.pct','sm__pipe_fma_cycles_active.avg.pct','sm__ops_path_tensor_op_utchmma_src_fp16_dst_fp32_sparsity_off.sum.pct','sm__pipe_tc_cycles_active.avg.pct']:
  for kk in h:
    if kk.startswith(k): print(kk, d[kk])
"
