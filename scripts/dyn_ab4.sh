cd $GRAFT_REPO_ROOT
export PYTHONPATH=$PWD
for d in 1 0 1 0; do BFPP_GEMM_DYN=$d timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline >> gpurun_out/r2_dyn_n1_$d.log 2>&1; echo "bench $d rc=$?"; done
