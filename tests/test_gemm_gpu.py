"""tcgen05 GEMM vs a plain PyTorch fp32 reference (bf16 inputs, f32 accumulate).

Tolerance: bf16 outputs -> max |err| <= 1e-2 * max|ref|; f32 outputs ->
1e-4 * max|ref| (accumulation-order differences only).
"""
import pytest
import torch

pytestmark = pytest.mark.gpu


def _ops():
    from paper_2211_05953_b200 import ops
    return ops


def _close(got, ref, rtol):
    err = (got.float() - ref).abs().max().item()
    scale = ref.abs().max().item() + 1e-6
    assert err <= rtol * scale, (err, scale)


# (mode, bn2, stream_k, dynamic): defaults (stream-K off); one-CTA tiles; two-CTA 256x128 and 256x256 pair
# tiles (forced), data-parallel and stream-K (forced: a k-split wherever every pair gets >= half a tile);
# the dynamic tile schedule (device counter + per-pair tile ring) with both pair-tile widths
VARIANTS = [(-1, 0, 0, 0), (-1, 0, -1, 0), (1, 0, 0, 0), (2, 128, 0, 0), (2, 256, 0, 0), (2, 256, 1, 0),
            (-1, 0, 0, 1), (2, 128, 0, 1)]


@pytest.fixture(params=VARIANTS, ids=lambda v: f"mode{v[0]}-bn{v[1]}-sk{v[2]}-dyn{v[3]}")
def variant(request, cuda_device):
    ops = _ops()
    ops.gemm_config(*request.param[:3])
    ops.gemm_schedule(bool(request.param[3]))
    yield request.param
    ops.gemm_config(-1, 0, 0)  # the library defaults
    ops.gemm_schedule(False)


@pytest.mark.parametrize("a_mn", [False, True])
@pytest.mark.parametrize("b_mn", [False, True])
@pytest.mark.parametrize("shape", [(256, 512, 128), (128, 256, 64), (384, 768, 320), (64, 1000, 128),
                                   (2048, 2048, 2048), (200, 136, 72), (512, 8192, 256), (2048, 8192, 2048),
                                   (768, 1280, 4096), (8448, 512, 4096)])  # last: N-fastest raster (A > 64 MB)
def test_gemm_layouts(variant, a_mn, b_mn, shape):
    ops = _ops()
    M, N, K = shape
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N + K)
    A = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    B = torch.randn(N, K, device="cuda", generator=g).bfloat16()
    ref = A.float() @ B.float().t()
    a_in = A.t().contiguous() if a_mn else A
    b_in = B.t().contiguous() if b_mn else B
    out = ops.gemm(a_in, b_in, a_mn_major=a_mn, b_mn_major=b_mn)
    torch.cuda.synchronize()
    _close(out, ref, 1e-2)
    out32 = ops.gemm(a_in, b_in, a_mn_major=a_mn, b_mn_major=b_mn, epilogue=ops.EPI_F32)
    torch.cuda.synchronize()
    _close(out32, ref, 1e-4)


def test_gemm_epilogues(variant):
    ops = _ops()
    M, N, K = 256, 768, 192
    A = torch.randn(M, K, device="cuda").bfloat16()
    B = (0.1 * torch.randn(N, K, device="cuda")).bfloat16()
    ref = A.float() @ B.float().t()
    pre = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    out = ops.gemm(A, B, epilogue=ops.EPI_GELU, aux_out=pre)
    _close(pre, ref, 1e-2)
    _close(out, torch.nn.functional.gelu(pre.float(), approximate="tanh"), 1e-2)
    R = torch.randn(M, N, device="cuda").bfloat16()
    out = ops.gemm(A, B, epilogue=ops.EPI_RESID, aux=R)
    _close(out, ref + R.float(), 1e-2)
    x = pre.float().requires_grad_()
    y = torch.nn.functional.gelu(x, approximate="tanh")
    (dg,) = torch.autograd.grad(y, x, torch.ones_like(y))
    out = ops.gemm(A, B, epilogue=ops.EPI_DGELU, aux=pre)
    _close(out, ref * dg, 1e-2)
    acc = torch.randn(M, N, device="cuda")
    base = acc.clone()
    ops.gemm(A, B, epilogue=ops.EPI_F32, out=acc, accumulate=True)
    torch.cuda.synchronize()
    _close(acc, base + ref, 1e-4)


def test_gemm_strided_views(cuda_device):
    """Leading dimensions larger than the logical width (e.g. Q/K/V slices of a fused QKV)."""
    ops = _ops()
    M, K = 256, 384
    X = torch.randn(M, 3 * K, device="cuda").bfloat16()
    W = torch.randn(512, K, device="cuda").bfloat16()
    view = X[:, K:2 * K]
    out = ops.gemm(view, W)
    _close(out, view.float() @ W.float().t(), 1e-2)


@pytest.mark.parametrize("shapes", [((512, 768, 256), (768, 512, 384)), ((2048, 2048, 512), (6144, 2048, 512)),
                                    ((256, 8192, 128), (8192, 256, 128))])
@pytest.mark.parametrize("epi", ["f32_acc", "bf16"])
@pytest.mark.parametrize("dyn", [False, True], ids=["static", "dynamic"])
def test_gemm_pair_matches_separate_launches(cuda_device, shapes, epi, dyn, request):
    """Grouped pair launch (one tile space) == two ordinary launches, bit for bit (same per-tile math),
    under the static and the dynamic tile schedule."""
    ops = _ops()
    ops.gemm_schedule(dyn)
    request.addfinalizer(lambda: ops.gemm_schedule(False))
    g = torch.Generator(device="cuda").manual_seed(11)
    probs = []
    for M, N, K in shapes:  # weight-gradient form: A = dY^T, B = X^T (both MN-major)
        A = torch.randn(K, M, device="cuda", generator=g).bfloat16()
        B = torch.randn(K, N, device="cuda", generator=g).bfloat16()
        probs.append((A, B, M, N))
    kw = dict(a_mn_major=True, b_mn_major=True)
    if epi == "f32_acc":
        kw.update(epilogue=ops.EPI_F32, accumulate=True)
        base = [torch.randn(M, N, device="cuda", generator=g) for _, _, M, N in probs]
    else:
        base = [torch.zeros(M, N, device="cuda", dtype=torch.bfloat16) for _, _, M, N in probs]
    sep = [b.clone() for b in base]
    grp = [b.clone() for b in base]
    for (A, B, _, _), o in zip(probs, sep):
        ops.gemm(A, B, out=o, **kw)
    ops.gemm_pair(dict(a=probs[0][0], b=probs[0][1], out=grp[0], **kw), dict(a=probs[1][0], b=probs[1][1], out=grp[1], **kw))
    torch.cuda.synchronize()
    for s_, g_, (A, B, _, _), b in zip(sep, grp, probs, base):
        assert torch.equal(s_, g_)
        ref = A.float().t() @ B.float() + (b.float() if epi == "f32_acc" else 0)
        _close(g_, ref, 1e-4 if epi == "f32_acc" else 1e-2)
