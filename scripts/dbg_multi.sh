export BFPP_HANG_DUMP_S=100
N=${N:-2}
for c in ${CASES}; do
mkdir -p gpurun_out/dbg/$c
timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=29611 tests/dist_worker.py --case $c --out gpurun_out/dbg/$c > gpurun_out/dbg/$c/log.txt 2>&1; echo "case $c rc=$?"
tail -5 gpurun_out/dbg/$c/log.txt
done
