# NCCL channel caps vs the GPT-1.3B N = 4 step (PP2 x 4 loops x DP2 DP_FS): fewer channels = fewer
# SMs taken from the compute stream by the all-gathers / reduce-scatters
cd $GRAFT_REPO_ROOT
for ch in default 2 4 8 16; do
  if [ $ch = default ]; then E=""; else E="NCCL_MAX_NCHANNELS=$ch NCCL_MIN_NCHANNELS=1"; fi
  env $E timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 \
    --master-port=$((29900 + RANDOM % 90)) bench.py --gpus 4 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline \
    > gpurun_out/r2_ch_$ch.log 2>&1
done
