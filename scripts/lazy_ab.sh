# lazy token-table update: executor parity, then the N = 1 step A/B and the per-task timeline
cd $GRAFT_REPO_ROOT
export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_executor_gpu.py -q -m gpu -x > gpurun_out/r2_lazy_exec.log 2>&1; echo "exec rc=$?"
for d in 1 0 1 0; do BFPP_LAZY_WTE=$d timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline >> gpurun_out/r2_lazy_n1_$d.log 2>&1; echo "bench $d rc=$?"; done
BFPP_LAZY_WTE=1 timeout 250 python scripts/timeline_probe.py > gpurun_out/r2_lazy_tl.log 2>&1
