# compute-sanitizer memcheck / racecheck / synccheck on the tcgen05 kernels at small shapes:
# attention fwd + bwd (2 x 256 x 3 heads: several query / key blocks, partial masks) and the
# 1-CTA / 2-CTA GEMMs with every epilogue, plus a grouped pair launch
cd $GRAFT_REPO_ROOT
CS=/usr/local/cuda/bin/compute-sanitizer
SEL="test_attention_fwd_bwd[2-256-3] or test_gemm_epilogues[mode1-bn0-sk0] or test_gemm_epilogues[mode2-bn256-sk0] or test_gemm_pair_matches_separate_launches[f32_acc-shapes0]"
for tool in memcheck racecheck synccheck; do
  timeout 1200 $CS --tool $tool --target-processes all --print-limit 20 \
    python -m pytest tests/test_kernels_gpu.py tests/test_gemm_gpu.py -m gpu -q -k "$SEL" -p no:cacheprovider \
    > gpurun_out/r2_sanitize_$tool.log 2>&1; echo rc=$? >> gpurun_out/r2_sanitize_$tool.log
done
