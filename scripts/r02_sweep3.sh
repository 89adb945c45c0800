# round-2 4-GPU evidence, part 3: the 52B layer shape (h 8192, 64 heads, seq 1024) at 16 layers,
# breadth-first PP2 x 4 loops x DP2 fully sharded with activation checkpoints, beta 1 and 2, vs
# depth-first and 1F1B; plan vs allocation in the bench line
cd $GRAFT_REPO_ROOT
for b in 1 2; do for s in breadth_first depth_first 1f1b; do
  l=4; [ $s = 1f1b ] && l=1
  timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 --master-port=$((29800 + b * 10 + l)) \
    bench.py --gpus 4 --model 52b-l16 --pp 2 --loops $l --beta $b --schedule $s --dp-variant dp_fs --recompute \
    --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02_52b_${s}_b$b.log 2>&1
done; done
