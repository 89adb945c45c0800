# dynamic vs static tile schedule of the 2-CTA GEMM: unit tests, per-CTA trace beside the
# optimizer, executor parity, N = 1 step both ways
cd $GRAFT_REPO_ROOT
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gemm_gpu.py -q -m gpu -x > gpurun_out/r2_dyn_gemm_tests.log 2>&1; echo "gemm tests rc=$?"
for s in "2048 8192 2048" "2048 6144 2048"; do echo "== $s"; timeout 100 python scripts/gemm_trace.py $s; done > gpurun_out/r2_dyn_trace.log 2>&1
timeout 900 python -m pytest tests/test_executor_gpu.py -q -m gpu -x > gpurun_out/r2_dyn_exec.log 2>&1; echo "exec rc=$?"
for d in 1 0 1 0; do BFPP_GEMM_DYN=$d timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline >> gpurun_out/r2_dyn_n1_$d.log 2>&1; echo "bench $d rc=$?"; done
BFPP_GEMM_DYN=1 timeout 300 python scripts/overlap_bench.py > gpurun_out/r2_dyn_overlap_1.log 2>&1
BFPP_GEMM_DYN=0 timeout 300 python scripts/overlap_bench.py > gpurun_out/r2_dyn_overlap_0.log 2>&1
