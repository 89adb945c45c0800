set -x
cd $GRAFT_REPO_ROOT
ncu --set full --import-source on --clock-control none -k regex:attn_bwd_tc2 -c 1 -o gpurun_out/attn_bwd2 python scripts/attn_bench.py 1 2048 16 > gpurun_out/ncu_attn1.log 2>&1
BFPP_ATTN_BWD=1 ncu --set full --import-source on --clock-control none -k regex:attn_bwd_tc_kernel -c 1 -o gpurun_out/attn_bwd1 python scripts/attn_bench.py 1 2048 16 >> gpurun_out/ncu_attn1.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:attn_fwd -c 1 -o gpurun_out/attn_fwd python scripts/attn_bench.py 1 2048 16 >> gpurun_out/ncu_attn1.log 2>&1
python scripts/attn_bench.py 1 2048 16 >> gpurun_out/ncu_attn1.log 2>&1
ls -la gpurun_out
