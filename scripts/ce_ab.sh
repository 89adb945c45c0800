# Copy-engine DP_FS all-gather (symmetric windows, CTAPolicy ZERO) vs the SM all-gather:
# multi-GPU parity first, then the N = 4 bench both ways (bench defaults: GPT-1.3B PP2 x 4 loops x DP2)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_multi_gpu.py -x -q -m gpu > gpurun_out/r2_ce_mgpu.log 2>&1; echo "mgpu rc=$?"
for ce in 1 0 1 0; do
  BFPP_DP_CE_ALLGATHER=$ce timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 \
    --master-port=$((29900 + RANDOM % 90)) bench.py --gpus 4 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline \
    >> gpurun_out/r2_ce_$ce.log 2>&1; echo "bench ce=$ce rc=$?"
done
