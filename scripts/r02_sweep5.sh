# GPT-13B (L32) PP4, 8 micro-batches, BF with 1 / 2 / 4 / 8 loops, with deferred weight gradients
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for l in 1 2 4 8; do timeout 600 python scripts/sweep.py --gpus 4 --model gpt-13b-l32 --pp 4 --loops $l --betas 2 --schedules breadth_first --dp-variant dp0 --out gpurun_out/r02_sweep_13b_defer.jsonl >> gpurun_out/r02_sweep_13b_defer.log 2>&1; echo "loops $l rc=$?"; done
