# bulk-staged LayerNorm kernels vs the register-resident ones: unit tests, isolated times, N = 1 step
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -m gpu -k "layernorm or ln" > gpurun_out/r2_ln_tests.log 2>&1; echo "tests rc=$?"
for b in 1 0; do BFPP_LN_BULK=$b timeout 300 python scripts/ln_bench.py > gpurun_out/r2_ln_bench_$b.log 2>&1; echo "ln_bench $b rc=$?"; done
timeout 900 python -m pytest tests/test_executor_gpu.py -q -m gpu -x > gpurun_out/r2_ln_exec.log 2>&1; echo "exec rc=$?"
for b in 1 0; do BFPP_LN_BULK=$b timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline >> gpurun_out/r2_ln_n1_$b.log 2>&1; echo "bench $b rc=$?"; done
