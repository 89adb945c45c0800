cd $GRAFT_REPO_ROOT
export PYTHONPATH=$PWD
for sms in 146 144; do echo "#### DYN=0 SMS=$sms"; for s in "2048 8192 2048" "2048 6144 2048"; do echo "== $s"; BFPP_GEMM_DYN=0 BFPP_GEMM_SMS=$sms timeout 100 python scripts/gemm_trace.py $s; done; done > gpurun_out/r2_dyn_trace5.log 2>&1
for v in "0 146" "0 0" "0 144" "0 146" "0 0"; do set -- $v; BFPP_GEMM_DYN=$1 BFPP_GEMM_SMS=$2 timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline >> gpurun_out/r2_sms_n1_$2.log 2>&1; echo "bench $v rc=$?"; done
