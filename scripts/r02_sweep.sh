# round-2 4-GPU evidence: GPT-6.7B BF vs DF vs 1F1B (PP4 x 2 loops, and PP2 x 4 loops x DP2 DP_FS),
# GPT-1.3B at N = 2 / 4 (weak scaling of BASELINE configs[1]), one recompute point
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python scripts/sweep.py --gpus 4 --model gpt-6.7b --pp 4 --loops 2 --betas 1 2 --schedules breadth_first depth_first 1f1b --dp-variant dp0 --out gpurun_out/r02_sweep_pp4.jsonl > gpurun_out/r02_sweep_pp4.log 2>&1
python scripts/sweep.py --gpus 4 --model gpt-6.7b --pp 2 --loops 4 --betas 1 2 --schedules breadth_first depth_first 1f1b --dp-variant dp_fs --out gpurun_out/r02_sweep_pp2dp2.jsonl > gpurun_out/r02_sweep_pp2dp2.log 2>&1
for n in 2 4; do timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr=127.0.0.1 --master-port=2950$n bench.py --gpus $n --steps 10 --warmup 3 > gpurun_out/r02_bench_n$n.log 2>&1; done
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 --master-port=29611 bench.py --gpus 4 --model gpt-6.7b --pp 2 --loops 4 --beta 2 --recompute --steps 6 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02_bench_6.7b_rc.log 2>&1
