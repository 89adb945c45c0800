export BFPP_HANG_DUMP_S=60
mkdir -p gpurun_out/dbg
for c in bf_pp2x2_mb4; do
timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29611 tests/dist_worker.py --case $c --out gpurun_out/dbg > gpurun_out/dbg/$c.log 2>&1; echo "case $c rc=$?"
tail -30 gpurun_out/dbg/$c.log
done
