cd $GRAFT_REPO_ROOT
for d in 0 1 0 1; do for n in 4 2; do
  BFPP_DEFER_WGRAD=$d timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr=127.0.0.1 \
    --master-port=$((29900 + RANDOM % 90)) bench.py --gpus $n --steps 30 --warmup 5 --no-e2e --no-cpu-baseline >> gpurun_out/r2_defer2_n${n}_$d.log 2>&1; echo "bench n=$n d=$d rc=$?"
done; done
