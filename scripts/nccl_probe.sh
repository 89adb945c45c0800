# NCCL settings vs the DP_FS all-gather / reduce-scatter rates inside the 6.7B PP2 x 4 loops x DP2 step
cd $GRAFT_REPO_ROOT
run() {
  tag=$1; shift
  env "$@" timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 \
    --master-port=$((29700 + RANDOM % 200)) bench.py --gpus 4 --model gpt-6.7b --pp 2 --loops 4 --beta 2 \
    --steps 6 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2_nccl_$tag.log 2>&1
}
run default
NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT,TUNING run debug NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT,TUNING
run ch32 NCCL_MIN_NCHANNELS=32
run nvls0 NCCL_NVLS_ENABLE=0
run ce NCCL_CTA_POLICY=1
