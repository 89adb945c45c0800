# dynamic vs static GEMM tile schedule at N = 4 (NCCL collectives hold SMs while GEMMs launch)
cd $GRAFT_REPO_ROOT
for d in 1 0 1 0; do
  BFPP_GEMM_DYN=$d timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 \
    --master-port=$((29900 + RANDOM % 90)) bench.py --gpus 4 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline >> gpurun_out/r2_dyn_n4_$d.log 2>&1; echo "bench d=$d rc=$?"
done
