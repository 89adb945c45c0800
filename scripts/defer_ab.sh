# deferred weight gradients: pipeline parity subset, then N = 2 / N = 4 bench A/B
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_multi_gpu.py -q -m gpu -k "tiny_bf_pp2x2_dp2_fs or small_bf_pp2x1 or 1f1b_pp2_mb4 or df_pp2x2_mb4 or steps3_small_bf_pp2x1_dp2_fs or bf_pp4x1_mb4" > gpurun_out/r2_defer_mgpu.log 2>&1; echo "mgpu rc=$?"
for d in 1 0 1 0; do for n in 4; do
  BFPP_DEFER_WGRAD=$d timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr=127.0.0.1 \
    --master-port=$((29900 + RANDOM % 90)) bench.py --gpus $n --steps 10 --warmup 3 --no-e2e --no-cpu-baseline >> gpurun_out/r2_defer_n${n}_$d.log 2>&1; echo "bench n=$n d=$d rc=$?"
done; done
for d in 1 0; do
  BFPP_DEFER_WGRAD=$d timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 \
    --master-port=$((29900 + RANDOM % 90)) bench.py --gpus 2 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline >> gpurun_out/r2_defer_n2_$d.log 2>&1; echo "bench n=2 d=$d rc=$?"
done
