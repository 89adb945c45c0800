#!/bin/bash
# Launch list + full captures of the top kernels of the N=1 bench (single GPU).
set -x
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-timeline"
timeout 300 $B > gpurun_out/plain.json 2> gpurun_out/plain.err; echo "plain rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_list.log 2>&1; echo "list rc=$?"
for k in gemm2_kernel attn_fwd_tc_kernel attn_bwd_tc_kernel ln_fwd_kernel ln_bwd_dx_kernel ln_bwd_param_kernel adam_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 20 -c 1 -o gpurun_out/full_$k -f $B > gpurun_out/ncu_$k.log 2>&1; echo "$k rc=$?"
done
