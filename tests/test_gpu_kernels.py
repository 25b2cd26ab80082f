"""Kernel-level numerics of libds on a B200: the tcgen05 GEMM in every operand
layout and the persistent recurrent kernels, each against a plain PyTorch
fp32 computation on the same bf16-rounded inputs.

Tolerances: the kernels accumulate in fp32 (TMEM) exactly like the torch
reference; differences come from summation order and fast sigmoid/tanh, so
fp32-level agreement is required for the GEMM (rel 1e-3) and bf16-ulp-level
agreement for values the kernels store as bf16.
"""

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1904_04956_b200 import _lib  # noqa: E402

DEV = "cuda:0"


def _gemm(a, a_mn, b, b_mn, M, N, K):
    lib = _lib.load()
    c = torch.zeros(M, N, device=DEV, dtype=torch.float32)
    rc = lib.ds_debug_gemm_bf16(
        a.data_ptr(), a.stride(0), a_mn, b.data_ptr(), b.stride(0), b_mn, c.data_ptr(), c.stride(0), M, N, K,
        _lib.stream_ptr(),
    )
    _lib.check(rc, "gemm")
    torch.cuda.synchronize()
    return c


@pytest.mark.parametrize("a_mn", [0, 1])
@pytest.mark.parametrize("b_mn", [0, 1])
@pytest.mark.parametrize("shape", [(256, 512, 128), (384, 768, 1024), (200, 272, 96), (4096, 1024, 5376)])
def test_gemm_layouts(a_mn, b_mn, shape):
    M, N, K = shape
    g = torch.Generator(device=DEV).manual_seed(M * 7 + N + K)
    A = torch.randn(M, K, device=DEV, generator=g).bfloat16()
    B = torch.randn(N, K, device=DEV, generator=g).bfloat16()
    a_store = A.t().contiguous() if a_mn else A
    b_store = B.t().contiguous() if b_mn else B
    C = _gemm(a_store, a_mn, b_store, b_mn, M, N, K)
    ref = A.float() @ B.float().t()
    err = (C - ref).abs().max().item()
    scale = ref.abs().max().item()
    assert err <= 1e-3 * scale + 1e-3, f"max err {err} (scale {scale})"


def _lstm_ref_fwd(G, W, B, T):
    H = 512
    N = T * B
    Y = torch.zeros(T, B, 2 * H, device=DEV)
    C = torch.zeros(T, B, 2 * H, device=DEV)
    A = torch.zeros(N, 8 * H, device=DEV)
    for d in range(2):
        Wd = W[d * 4 * H:(d + 1) * 4 * H].float()
        h = torch.zeros(B, H, device=DEV)
        c = torch.zeros(B, H, device=DEV)
        order = range(T) if d == 0 else range(T - 1, -1, -1)
        for t in order:
            a = G[t * B:(t + 1) * B, d * 4 * H:(d + 1) * 4 * H].float() + h @ Wd.t()
            a = a.view(B, H, 4)
            i, f, gg, o = a[..., 0].sigmoid(), a[..., 1].sigmoid(), a[..., 2].tanh(), a[..., 3].sigmoid()
            c = f * c + i * gg
            hh = o * c.tanh()
            h = hh.bfloat16().float()
            Y[t, :, d * H:(d + 1) * H] = h
            C[t, :, d * H:(d + 1) * H] = c
            A[t * B:(t + 1) * B, d * 4 * H:(d + 1) * 4 * H] = torch.stack([i, f, gg, o], -1).view(B, 4 * H)
    return Y, C, A


def _lstm_ref_bwd(acts, C, dY, WT, B, T):
    H = 512
    N = T * B
    dG = torch.zeros(N, 8 * H, device=DEV)
    Cv = C.view(T, B, 2 * H)
    for d in range(2):
        WdT = WT[d * H:(d + 1) * H].float()  # [512, 2048]
        dh_rec = torch.zeros(B, H, device=DEV)
        dcc = torch.zeros(B, H, device=DEV)
        order = range(T - 1, -1, -1) if d == 0 else range(T)
        for t in order:
            rows = slice(t * B, (t + 1) * B)
            dh = dh_rec + dY[rows, d * H:(d + 1) * H].float()
            a = acts[rows, d * 4 * H:(d + 1) * 4 * H].float().view(B, H, 4)
            i, f, gg, o = a[..., 0], a[..., 1], a[..., 2], a[..., 3]
            c = Cv[t, :, d * H:(d + 1) * H]
            tp = t - 1 if d == 0 else t + 1
            cp = Cv[tp, :, d * H:(d + 1) * H] if 0 <= tp < T else torch.zeros_like(c)
            tc = c.tanh()
            dc = dh * o * (1 - tc * tc) + dcc
            dgi = dc * gg * i * (1 - i)
            dgf = dc * cp * f * (1 - f)
            dgg = dc * i * (1 - gg * gg)
            dgo = dh * tc * o * (1 - o)
            dcc = dc * f
            dg = torch.stack([dgi, dgf, dgg, dgo], -1).view(B, 4 * H).bfloat16().float()
            dG[rows, d * 4 * H:(d + 1) * 4 * H] = dg
            dh_rec = dg @ WdT.t()
    return dG


@pytest.mark.parametrize("B,T", [(160, 6), (256, 21), (600, 3)])
def test_lstm_recurrent_fwd_bwd(B, T):
    lib = _lib.load()
    H = 512
    N = T * B
    g = torch.Generator(device=DEV).manual_seed(B + T)
    G = (torch.randn(N, 8 * H, device=DEV, generator=g) * 0.5).bfloat16()
    W = (torch.randn(8 * H, H, device=DEV, generator=g) * 0.05).bfloat16()
    WT = torch.cat([W[:4 * H].t(), W[4 * H:].t()], 0).contiguous()  # [1024, 2048]
    gates = G.clone()
    cstate = torch.zeros(N, 2 * H, device=DEV)
    yfull = torch.zeros((T + 2) * B, 2 * H, device=DEV, dtype=torch.bfloat16)
    counters = torch.zeros(16384, device=DEV, dtype=torch.int32)
    rc = lib.ds_debug_lstm_fwd(B, T, gates.data_ptr(), cstate.data_ptr(), yfull.data_ptr(), W.data_ptr(),
                               counters.data_ptr(), None, _lib.stream_ptr())
    _lib.check(rc, "lstm_fwd")
    torch.cuda.synchronize()
    Y, C, A = _lstm_ref_fwd(G, W, B, T)
    y_k = yfull[B:(T + 1) * B].float().view(T, B, 2 * H)
    assert (y_k - Y).abs().max().item() < 2e-2
    assert (cstate.view(T, B, 2 * H) - C).abs().max().item() < 2e-2
    assert (gates.float() - A).abs().max().item() < 1e-2
    # padding rows stay zero
    assert yfull[:B].abs().max().item() == 0 and yfull[(T + 1) * B:].abs().max().item() == 0

    dY = torch.randn(N, 2 * H, device=DEV, generator=g).bfloat16()
    dg = torch.zeros(N, 8 * H, device=DEV, dtype=torch.bfloat16)
    rc = lib.ds_debug_lstm_bwd(B, T, gates.data_ptr(), cstate.data_ptr(), W.data_ptr(), dY.data_ptr(),
                               dg.data_ptr(), counters.data_ptr(), None, _lib.stream_ptr())
    _lib.check(rc, "lstm_bwd")
    torch.cuda.synchronize()
    ref = _lstm_ref_bwd(gates, cstate, dY, WT, B, T)
    err = (dg.float() - ref).abs().max().item()
    scale = ref.abs().max().item()
    assert err <= 2e-2 * scale, f"dG err {err} scale {scale}"


@pytest.mark.timeout(300)
def test_lstm_back_to_back_launches_reuse_flags():
    """The recurrent kernels' step flags count up across launches (no reset): a
    second, third, ... launch on the same counters, issued back to back under
    programmatic dependent launch, must neither hang nor change the result."""
    lib = _lib.load()
    H, B, T = 512, 256, 5
    N = T * B
    g = torch.Generator(device=DEV).manual_seed(7)
    G = (torch.randn(N, 8 * H, device=DEV, generator=g) * 0.5).bfloat16()
    W = (torch.randn(8 * H, H, device=DEV, generator=g) * 0.05).bfloat16()
    dY = torch.randn(N, 2 * H, device=DEV, generator=g).bfloat16()
    counters = torch.zeros(16384, device=DEV, dtype=torch.int32)
    outs = []
    for _ in range(3):
        gates = G.clone()
        cstate = torch.zeros(N, 2 * H, device=DEV)
        yfull = torch.zeros((T + 2) * B, 2 * H, device=DEV, dtype=torch.bfloat16)
        dg = torch.zeros(N, 8 * H, device=DEV, dtype=torch.bfloat16)
        s = _lib.stream_ptr()
        for _ in range(2):  # two forward launches, then two backward launches, nothing in between
            _lib.check(lib.ds_debug_lstm_fwd(B, T, gates.data_ptr(), cstate.data_ptr(), yfull.data_ptr(), W.data_ptr(),
                                             counters.data_ptr(), None, s), "lstm_fwd")
        for _ in range(2):
            _lib.check(lib.ds_debug_lstm_bwd(B, T, gates.data_ptr(), cstate.data_ptr(), W.data_ptr(), dY.data_ptr(),
                                             dg.data_ptr(), counters.data_ptr(), None, s), "lstm_bwd")
        torch.cuda.synchronize()
        outs.append((yfull.clone(), cstate.clone(), dg.clone()))
    for o in outs[1:]:
        for a, b in zip(outs[0], o):
            assert torch.equal(a, b)
