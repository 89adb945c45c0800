# GEMM pipeline depth vs optimizer co-running: overlap_bench and the N = 1 step with the default
# 5-stage library and 4 / 6-stage builds (libbfpp_s4.so / libbfpp_s6.so, -DBFPP_GEMM2_STAGES=n)
cd $GRAFT_REPO_ROOT
export PYTHONPATH=$PWD
for lib in libbfpp.so libbfpp_s6.so libbfpp.so libbfpp_s6.so; do echo "== $lib"; BFPP_LIB_PATH=$PWD/paper_2211_05953_b200/$lib timeout 200 python scripts/overlap_bench.py 2>&1 | head -2; done > gpurun_out/r2_gemm_stages6.log
for lib in libbfpp.so libbfpp_s6.so libbfpp.so libbfpp_s6.so; do BFPP_LIB_PATH=$PWD/paper_2211_05953_b200/$lib timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline >> gpurun_out/r2_stages_n1_$lib.log 2>&1; echo "bench $lib rc=$?"; done
