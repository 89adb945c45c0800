# GEMM pipeline depth vs optimizer co-running: overlap_bench with the default 5-stage library and
# a 4-stage build (paper_2211_05953_b200/libbfpp_s4.so, -DBFPP_GEMM2_STAGES=4)
cd $GRAFT_REPO_ROOT
export PYTHONPATH=$PWD
for lib in libbfpp.so libbfpp_s4.so libbfpp.so libbfpp_s4.so; do echo "== $lib"; BFPP_LIB_PATH=$PWD/paper_2211_05953_b200/$lib timeout 200 python scripts/overlap_bench.py 2>&1 | head -2; done > gpurun_out/r2_gemm_stages.log
