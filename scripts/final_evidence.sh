#!/bin/bash
# Round-end evidence on one B200 (single GPU; ncu only after the same command exited 0):
# smoke, the default bench line, the ncu launch list with DRAM bytes, full captures of the top kernels.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/gputest_1gpu.log 2>&1; echo "gputest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 400 python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; echo "bench rc=$?"
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-timeline"
timeout 300 $B > gpurun_out/plain.json 2> gpurun_out/plain.err; echo "plain rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_list.log 2>&1; echo "list rc=$?"
for k in gemm2_kernel attn_fwd_tc_kernel attn_bwd_tc_kernel ln_bwd_bulk_kernel ln_fwd_reg_kernel adam_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 20 -c 1 -o gpurun_out/full_$k -f $B \
    > gpurun_out/ncu_$k.log 2>&1; echo "$k rc=$?"
done
# GPT-6.7B on one B200 (no pipeline bubble: the per-GPU efficiency ceiling of the 6.7B shapes)
for b in 1 2; do
  timeout 600 python bench.py --model gpt-6.7b --loops 4 --beta $b --steps 5 --warmup 3 --no-e2e --no-cpu-baseline \
    > gpurun_out/bench_6.7b_n1_b$b.json 2> gpurun_out/bench_6.7b_n1_b$b.err; echo "6.7b b$b rc=$?"
done
