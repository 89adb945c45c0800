cd $GRAFT_REPO_ROOT
export PYTHONPATH=$PWD
for d in 1 0; do echo "#### DYN=$d"; for s in "2048 8192 2048" "2048 6144 2048"; do echo "== $s"; BFPP_GEMM_DYN=$d timeout 100 python scripts/gemm_trace.py $s; done; done > gpurun_out/r2_dyn_trace.log 2>&1
for d in 1 0 1 0; do BFPP_GEMM_DYN=$d timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline >> gpurun_out/r2_dyn_n1_$d.log 2>&1; echo "bench $d rc=$?"; done
