# Adam grid cap vs GEMM co-running slowdown (scripts/overlap_bench.py), then the N = 1 step
cd $GRAFT_REPO_ROOT
export PYTHONPATH=$PWD
for g in 0 592 296 148 74; do echo "== BFPP_ADAM_GRID=$g"; BFPP_ADAM_GRID=$g timeout 200 python scripts/overlap_bench.py 2>&1 | head -3; done > gpurun_out/r2_adam_pace.log
for g in 0 296 148; do BFPP_ADAM_GRID=$g timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r2_adam_pace_n1_$g.log 2>&1; done
