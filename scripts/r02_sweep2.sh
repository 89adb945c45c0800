# round-2 4-GPU evidence, part 2: GPT-13B (L32 h5760) PP4, 8 micro-batches of 1 sequence, bubble vs
# loop count (BASELINE configs[3] on 4 GPUs); GPT-1.3B N = 4 with the per-task replay bubble
cd $GRAFT_REPO_ROOT
python scripts/sweep.py --gpus 4 --model gpt-13b-l32 --pp 4 --loops 1 --betas 2 --schedules breadth_first --dp-variant dp0 --out gpurun_out/r02_sweep_13b.jsonl > gpurun_out/r02_sweep_13b.log 2>&1
for l in 2 4 8; do python scripts/sweep.py --gpus 4 --model gpt-13b-l32 --pp 4 --loops $l --betas 2 --schedules breadth_first --dp-variant dp0 --out gpurun_out/r02_sweep_13b.jsonl >> gpurun_out/r02_sweep_13b.log 2>&1; done
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 --master-port=29514 bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/r02_bench_n4b.log 2>&1
