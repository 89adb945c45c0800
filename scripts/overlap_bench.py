"""GEMM (high-priority stream) vs Adam (low-priority stream) co-running: does the optimizer
stream HBM under tensor-core work? Prints each side alone and together."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_05953_b200 import ops  # noqa: E402

T, h = 2048, 2048
m = 4 * h
E = ops
shapes = [(T, 3 * h, h, 0, 0, E.EPI_BF16), (T, h, h, 0, 0, E.EPI_RESID), (T, m, h, 0, 0, E.EPI_GELU),
          (T, h, m, 0, 0, E.EPI_RESID), (h, m, T, 1, 1, E.EPI_F32), (T, m, h, 0, 1, E.EPI_DGELU),
          (m, h, T, 1, 1, E.EPI_F32), (T, h, m, 0, 1, E.EPI_BF16), (h, h, T, 1, 1, E.EPI_F32),
          (T, h, h, 0, 1, E.EPI_BF16), (3 * h, h, T, 1, 1, E.EPI_F32), (T, h, 3 * h, 0, 1, E.EPI_BF16)]
bufs = []
for M, N, K, amn, bmn, epi in shapes:
    a = torch.randn((K, M) if amn else (M, K), device="cuda").to(torch.bfloat16)
    b = torch.randn((K, N) if bmn else (N, K), device="cuda").to(torch.bfloat16)
    out = torch.empty(M, N, device="cuda", dtype=torch.float32 if epi == E.EPI_F32 else torch.bfloat16)
    aux = torch.randn(M, N, device="cuda").to(torch.bfloat16) if epi in (E.EPI_RESID, E.EPI_DGELU) else None
    aux_out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16) if epi == E.EPI_GELU else None
    bufs.append((a, b, amn, bmn, out, epi, aux, aux_out))
flops_layer = sum(2.0 * M * N * K for M, N, K, *_ in shapes)
n_param = int(os.environ.get("NPARAM", str(300 << 20)))
p = torch.randn(n_param, device="cuda")
mm, vv, g = torch.zeros_like(p), torch.ones_like(p), torch.randn_like(p)
w16 = torch.empty(n_param, device="cuda", dtype=torch.bfloat16)
hi = torch.cuda.Stream(priority=-5)
lo = torch.cuda.Stream(priority=0)
LAYERS = int(os.environ.get("LAYERS", "24"))


def gemms():
    for _ in range(LAYERS):
        for a, b, amn, bmn, out, epi, aux, aux_out in bufs:
            ops.gemm(a, b, a_mn_major=bool(amn), b_mn_major=bool(bmn), out=out, epilogue=epi, aux=aux,
                     aux_out=aux_out)


def adam(k):
    for _ in range(k):
        ops.adam_update_(p, mm, vv, g, w16, 1e-4, 0.9, 0.95, 1e-8, 0.0, 1)


def timed(run_g, run_a, k):
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    with torch.cuda.stream(hi):
        ev[0].record()
    lo.wait_stream(hi)
    if run_g:
        with torch.cuda.stream(hi):
            gemms()
    with torch.cuda.stream(hi):
        ev[1].record()
    with torch.cuda.stream(lo):
        ev[2].record()
        if run_a:
            adam(k)
        ev[3].record()
    torch.cuda.synchronize()
    return ev[0].elapsed_time(ev[1]), ev[2].elapsed_time(ev[3])


for _ in range(2):
    timed(True, True, 1)
g_alone, _ = timed(True, False, 0)
_, a_alone = timed(False, True, 1)
k = max(1, int(g_alone / a_alone))
g_both, a_both = timed(True, True, k)
print(f"gemm alone {g_alone:.2f} ms ({flops_layer * LAYERS / g_alone / 1e9:.0f} TF/s); "
      f"adam alone {a_alone:.2f} ms ({30.0 * n_param / a_alone / 1e6:.0f} GB/s)")
print(f"together (adam x{k}): gemm {g_both:.2f} ms ({flops_layer * LAYERS / g_both / 1e9:.0f} TF/s), "
      f"adam {a_both:.2f} ms ({30.0 * n_param * k / a_both / 1e6:.0f} GB/s)")


# ---- SM partition (green contexts): GEMM stream on N - k SMs, optimizer stream on k SMs ----
def green_streams(k):
    """Two CUDA streams confined to disjoint SM partitions of the current device (k SMs for the
    second). Returns (big_stream, small_stream, n_big) or None when unsupported."""
    from cuda.bindings import driver as d
    dev = torch.cuda.current_device()
    err, cudev = d.cuDeviceGet(dev)
    err, res = d.cuDeviceGetDevResource(cudev, d.CUdevResourceType.CU_DEV_RESOURCE_TYPE_SM)
    if err != d.CUresult.CUDA_SUCCESS:
        return None
    total = res.sm.smCount
    # split off groups of k SMs: the first group goes to the optimizer, the remainder to the GEMMs
    err, groups, n, rem = d.cuDevSmResourceSplitByCount(1, res, 0, k)
    if err != d.CUresult.CUDA_SUCCESS:
        print("split failed", err)
        return None
    out = []
    for r in (rem, groups[0]):
        err, desc = d.cuDevResourceGenerateDesc([r], 1)
        err, gctx = d.cuGreenCtxCreate(desc, cudev, d.CUgreenCtxCreate_flags.CU_GREEN_CTX_DEFAULT_STREAM)
        err, s = d.cuGreenCtxStreamCreate(gctx, d.CUstream_flags.CU_STREAM_NON_BLOCKING, 0)
        out.append((int(s), r.sm.smCount))
    print(f"partition: {out[0][1]} SMs (GEMM) + {out[1][1]} SMs (optimizer) of {total}")
    return out


if os.environ.get("GREEN_SPLIT"):
    from paper_2211_05953_b200 import _native as NAT
    for k in [int(x) for x in os.environ["GREEN_SPLIT"].split(",")]:
        gs = green_streams(k)
        if gs is None:
            print("green contexts unavailable")
            break
        (sb, nb), (ss, ns) = gs
        NAT.lib().bfpp_gemm_sm_limit(nb)
        hi = torch.cuda.ExternalStream(sb)
        lo = torch.cuda.ExternalStream(ss)
        for _ in range(2):
            timed(True, True, 1)
        g_alone, _ = timed(True, False, 0)
        _, a_alone = timed(False, True, 1)
        kk = max(1, int(g_alone / a_alone))
        g_both, a_both = timed(True, True, kk)
        print(f"[{nb}+{ns} SMs] gemm alone {g_alone:.2f} ms ({flops_layer * LAYERS / g_alone / 1e9:.0f} TF/s); "
              f"adam alone {a_alone:.2f} ms ({30.0 * n_param / a_alone / 1e6:.0f} GB/s); together (adam x{kk}): "
              f"gemm {g_both:.2f} ms ({flops_layer * LAYERS / g_both / 1e9:.0f} TF/s), "
              f"adam {a_both:.2f} ms ({30.0 * n_param * kk / a_both / 1e6:.0f} GB/s)")
        NAT.lib().bfpp_gemm_sm_limit(0)
