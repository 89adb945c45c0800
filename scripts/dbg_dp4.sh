# repeats the DP4 / DP2 fully sharded breadth-first parity cases (race hunting)
cd $GRAFT_REPO_ROOT
for i in 1 2 3; do timeout 300 python -m pytest tests/test_multi_gpu.py -m gpu -q -k "bf_pp1x2_dp4_fs or bf_pp1x4_dp2_fs or steps3_tiny_bf_pp2x2_dp2_fs_rc" > gpurun_out/r2_dbg_$i.log 2>&1; echo rc=$? >> gpurun_out/r2_dbg_$i.log; done
