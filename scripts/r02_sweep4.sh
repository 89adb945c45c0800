# GPT-6.7B BF vs DF vs 1F1B at beta = 2 with deferred weight gradients (PP4 x 2 loops DP1; PP2 x 4 loops x DP2 DP_FS)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python scripts/sweep.py --gpus 4 --model gpt-6.7b --pp 2 --loops 4 --betas 2 --schedules breadth_first depth_first 1f1b --dp-variant dp_fs --out gpurun_out/r02_sweep_pp2dp2_defer.jsonl > gpurun_out/r02_sweep_pp2dp2_defer.log 2>&1; echo "pp2dp2 rc=$?"
python scripts/sweep.py --gpus 4 --model gpt-6.7b --pp 4 --loops 2 --betas 2 --schedules breadth_first depth_first 1f1b --dp-variant dp0 --out gpurun_out/r02_sweep_pp4_defer.jsonl > gpurun_out/r02_sweep_pp4_defer.log 2>&1; echo "pp4 rc=$?"
