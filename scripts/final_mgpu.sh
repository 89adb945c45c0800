# Round-end multi-GPU evidence on 4 B200s: multi-GPU parity, then the N = 2 and N = 4 bench lines
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_multi_gpu.py -q -m gpu > gpurun_out/mgpu_final.log 2>&1; echo "mgpu rc=$?"
for n in 2 4; do
  timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr=127.0.0.1 \
    --master-port=$((29900 + RANDOM % 90)) bench.py --gpus $n > gpurun_out/bench_n$n.log 2>&1; echo "bench n=$n rc=$?"
done
