cd $GRAFT_REPO_ROOT
export PYTHONPATH=$PWD
for d in 2 1 0; do echo "#### DYN=$d"; for s in "2048 8192 2048"; do echo "== $s"; BFPP_GEMM_DYN=$d timeout 100 python scripts/gemm_trace.py $s; done; done > gpurun_out/r2_dyn_trace3.log 2>&1
