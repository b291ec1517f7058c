"""Kernel-level parity on the B200 (through the C-ABI).

* projection GEMM (tcgen05 and SIMT) vs an fp32 torch reference of the same op
* K10 shuffle vs a torch slice-copy reference -- bit exact
"""

import ctypes as C

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from paper_2305_13484_b200 import _lib  # noqa: E402

EPI_STORE, EPI_GELU, EPI_ACC, EPI_F32 = 0, 1, 2, 3


def _gelu(x):
    return 0.5 * x * (1.0 + torch.tanh(0.7978845608028654 * (x + 0.044715 * x ** 3)))


class _Tiled:
    """A tiled weight buffer with the logical [N, K] shape (for _gemm)."""

    def __init__(self, t, n, k):
        self.t, self.shape = t, (n, k)

    def data_ptr(self):
        return self.t.data_ptr()


def _gemm(x, w, bias, out, epi, use_tc, dtype):
    lib = _lib.load()
    ws = torch.empty(lib.fl_gemm_workspace_bytes(), dtype=torch.uint8, device="cuda")
    M, K = x.shape
    N = w.shape[0]
    s = torch.cuda.current_stream()
    _lib.check(lib.fl_gemm(x.data_ptr(), x.stride(0), w.data_ptr(),
                           bias.data_ptr() if bias is not None else None, out.data_ptr(),
                           out.stride(0), M, N, K, epi, dtype, int(use_tc), ws.data_ptr(),
                           C.c_void_p(s.cuda_stream)))
    torch.cuda.synchronize()
    return ws


SHAPES = [(1, 768, 768), (7, 2304, 768), (16, 512, 1024), (55, 3072, 768), (64, 768, 3072),
          (100, 50257, 768), (129, 1536, 4096), (256, 4096, 512), (300, 1000, 256), (17, 128, 64),
          (350, 1536, 4096), (512, 768, 768), (700, 1024, 512), (1000, 384, 256),
          # GPT-J 6B projection shapes at a saturated window (stream-K splits tiles)
          (320, 12288, 4096), (262, 4096, 16384), (96, 16384, 4096), (5, 4096, 4096),
          # more 256-row tiles than SM pairs at >= 128 rows: ranges of tpr >= 2
          # whole tiles (GPT-J merged QKV + FFN-up, NeoX merged, LM head)
          (192, 28672, 4096), (136, 30720, 6144), (320, 50400, 4096)]


@pytest.mark.parametrize("M,N,K", SHAPES)
@pytest.mark.parametrize("epi", [EPI_STORE, EPI_GELU, EPI_ACC, EPI_F32])
def test_tcgen05_gemm_matches_fp32_reference(M, N, K, epi):
    g = torch.Generator(device="cuda").manual_seed(M * 131 + N * 7 + K)
    x = (torch.randn(M, K, device="cuda", generator=g) * 0.5).bfloat16()
    w = (torch.randn(N, K, device="cuda", generator=g) * 0.05).bfloat16()
    b = (torch.randn(N, device="cuda", generator=g) * 0.1).bfloat16()
    ref = x.float() @ w.float().T + b.float()
    if epi in (EPI_STORE, EPI_GELU):
        out = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
        if epi == EPI_GELU:
            ref = _gelu(ref)
    else:
        out = torch.randn(M, N, device="cuda", generator=g)
        if epi == EPI_ACC:
            ref = ref + out
    _gemm(x, w, b, out, epi, True, 1)
    # fp32 accumulation of bf16 products: error ~ sqrt(K) * 2^-9 * |x||w|;
    # bf16 outputs add one rounding (2^-8 relative)
    tol = 2e-3 * (K / 256) ** 0.5 + (2.0 ** -8) * ref.abs().max().item() * (epi in (0, 1))
    err = (out.float() - ref).abs().max().item()
    assert err <= tol, (err, tol)


@pytest.mark.parametrize("M,N,K", [(1, 256, 256), (33, 1000, 512), (70, 768, 3072)])
def test_simt_gemm_fp32_matches_reference(M, N, K):
    g = torch.Generator(device="cuda").manual_seed(5)
    x = torch.randn(M, K, device="cuda", generator=g)
    w = torch.randn(N, K, device="cuda", generator=g) * 0.05
    b = torch.randn(N, device="cuda", generator=g)
    out = torch.empty(M, N, device="cuda")
    _gemm(x, w, b, out, EPI_F32, False, 0)
    ref = (x.double() @ w.double().T + b.double()).float()
    assert (out - ref).abs().max().item() < 1e-4 * (K / 256) ** 0.5


def test_tcgen05_split_k_counters_self_reset():
    """Two identical split-K GEMMs through one workspace give identical results."""
    x = torch.randn(3, 4096, device="cuda").bfloat16()
    w = (torch.randn(512, 4096, device="cuda") * 0.02).bfloat16()
    o1 = torch.empty(3, 512, device="cuda")
    o2 = torch.empty(3, 512, device="cuda")
    _gemm(x, w, None, o1, EPI_F32, True, 1)
    _gemm(x, w, None, o2, EPI_F32, True, 1)
    assert torch.equal(o1, o2)


def test_shuffle_kernel_bit_exact():
    from paper_2305_13484_b200.executor import CudaExecutor
    from paper_2305_13484_b200.models import get_spec
    spec = get_spec("gpt2-mini")
    ex = CudaExecutor(spec, {}, dtype="bf16", pool_slots=8, max_seq=40, max_new_tokens=8)
    ex.kv.copy_(torch.randn_like(ex.kv, dtype=torch.float32).bfloat16())
    before = ex.kv.clone()
    moves = [(6, 1, 33), (7, 2, 5), (0, 3, 40)]
    flat = (C.c_int32 * 9)(*[v for m in moves for v in m])
    _lib.check(ex.lib.fl_shuffle(ex.handle, flat, 3, C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    torch.cuda.synchronize()
    ref = before.clone()
    for s, d, n in moves:
        ref[:, d, :, :, :n] = before[:, s, :, :, :n]
    assert torch.equal(ex.kv, ref)
    ex.close()


@pytest.mark.parametrize("M,N,K", [(8, 12288, 4096), (320, 12288, 4096), (262, 4096, 16384), (100, 50257, 768),
                                   (300, 1000, 256), (700, 1024, 512), (129, 1536, 4096),
                                   (192, 28672, 4096), (136, 30720, 6144)])
@pytest.mark.parametrize("epi", [EPI_STORE, EPI_ACC])
def test_tcgen05_gemm_tiled_weights(M, N, K, epi):
    """fl_tile_weight layout ([N/128][K/64][128][64]) + use_tc = 2 gives the
    same result as the row-major weights (bit-identical accumulation order)."""
    lib = _lib.load()
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    x = (torch.randn(M, K, device="cuda", generator=g) * 0.5).bfloat16()
    w = (torch.randn(N, K, device="cuda", generator=g) * 0.05).bfloat16()
    b = (torch.randn(N, device="cuda", generator=g) * 0.1).bfloat16()
    wt = torch.empty(lib.fl_tiled_weight_bytes(N, K) // 2, dtype=torch.bfloat16, device="cuda")
    _lib.check(lib.fl_tile_weight(w.data_ptr(), N, K, wt.data_ptr(), C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    if epi == EPI_STORE:
        o1 = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
    else:
        o1 = torch.randn(M, N, device="cuda", generator=g)
    o2 = o1.clone()
    _gemm(x, w, b, o1, epi, 1, 1)
    _gemm(x, _Tiled(wt, N, K), b, o2, epi, 2, 1)
    if epi == EPI_STORE:
        assert torch.equal(o1, o2)
    else:
        assert (o1 - o2).abs().max().item() <= 1e-4 * o1.abs().max().item()


@pytest.mark.parametrize("hd", [64, 96, 128, 256])
@pytest.mark.parametrize("M,Hl", [(3, 4), (40, 8), (150, 2)])
def test_attention_kernel_matches_fp32_reference(hd, M, Hl):
    """K4 through the C-ABI (fl_attention) against a plain torch fp32 softmax
    attention over each row's own slot and context (1 <= ctx <= S, ragged;
    split-K + combine at small M * Hl, single pass at large)."""
    import ctypes as C
    from paper_2305_13484_b200 import _lib
    lib = _lib.load()
    S = 700
    Cs = M + 3
    g = torch.Generator(device="cuda").manual_seed(hd * 1000 + M)
    kv = torch.randn(Cs, 2, Hl, S, hd, device="cuda", generator=g).bfloat16()
    q = torch.randn(M, Hl * hd, device="cuda", generator=g).bfloat16()
    ctx = torch.randint(1, S + 1, (M,), device="cuda", generator=g, dtype=torch.int32)
    ctx[0] = 1
    ctx[-1] = S
    slots = torch.randperm(Cs, device="cuda", generator=g)[:M].to(torch.int32)
    rows = torch.zeros(M, 6, dtype=torch.int32, device="cuda")
    rows[:, 0] = slots
    rows[:, 1] = torch.arange(M, dtype=torch.int32, device="cuda")
    rows[:, 2] = ctx - 1
    rows[:, 4] = _lib.ROW_DECODE
    ws = torch.empty(lib.fl_attention_workspace_bytes(M, Hl, hd, S), dtype=torch.uint8, device="cuda")
    out = torch.empty(M, Hl * hd, dtype=torch.bfloat16, device="cuda")
    _lib.check(lib.fl_attention(q.data_ptr(), rows.data_ptr(), ctx.data_ptr(), M, Hl, hd, kv.data_ptr(), Cs, S,
                                out.data_ptr(), ws.data_ptr(), _lib.FL_DTYPE["bf16"],
                                C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    torch.cuda.synchronize()
    ref = torch.empty(M, Hl, hd, device="cuda")
    qf = q.float().view(M, Hl, hd)
    for r in range(M):
        n = int(ctx[r])
        k = kv[int(slots[r]), 0, :, :n].float()          # [Hl, n, hd]
        v = kv[int(slots[r]), 1, :, :n].float()
        p = torch.softmax(torch.einsum("hd,hnd->hn", qf[r], k) / hd ** 0.5, dim=-1)
        ref[r] = torch.einsum("hn,hnd->hd", p, v)
    torch.testing.assert_close(out.float().view(M, Hl, hd), ref, atol=2e-2, rtol=2e-2)


def _gemm2(x, x2, w, bias, out, epi, use_tc, nsplit=0, ogap=0, keys=None, index_base=0, N=None, K=None):
    lib = _lib.load()
    ws = torch.empty(lib.fl_gemm_workspace_bytes(), dtype=torch.uint8, device="cuda")
    M = x.shape[0]
    N = N or w.shape[0]
    K = K or x.shape[1]
    s = torch.cuda.current_stream()
    _lib.check(lib.fl_gemm2(x.data_ptr(), x2.data_ptr() if x2 is not None else None, x.stride(0),
                            w.data_ptr(), bias.data_ptr() if bias is not None else None,
                            out.data_ptr() if out is not None else None, out.stride(0) if out is not None else 0,
                            M, N, K, epi, 1, use_tc, nsplit, ogap,
                            keys.data_ptr() if keys is not None else None, index_base, ws.data_ptr(),
                            C.c_void_p(s.cuda_stream)))
    torch.cuda.synchronize()


def _tile(w):
    lib = _lib.load()
    n, k = w.shape
    wt = torch.empty(lib.fl_tiled_weight_bytes(n, k) // 2, dtype=torch.bfloat16, device="cuda")
    _lib.check(lib.fl_tile_weight(w.data_ptr(), n, k, wt.data_ptr(), C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    return wt


@pytest.mark.parametrize("M", [8, 40, 96, 136, 192, 256, 320])
@pytest.mark.parametrize("tiled", [False, True])
def test_dual_gemm_merged_in_projection(M, tiled):
    """fl_set_merged_in's GEMM at the GPT-J shape: [W_qkv; W_fc] (12288 +
    16384 rows, K 4096) in one launch; rows < 12288 read x and store into
    columns [0, 12288), rows >= 12288 read x2, get GELU and land at column
    n + 4096 of the shared [M][4Dl + Fl] activation row."""
    d, q3, F = 4096, 12288, 16384
    g = torch.Generator(device="cuda").manual_seed(M)
    x = (torch.randn(M, d, device="cuda", generator=g) * 0.5).bfloat16()
    x2 = (torch.randn(M, d, device="cuda", generator=g) * 0.5).bfloat16()
    w = (torch.randn(q3 + F, d, device="cuda", generator=g) * 0.02).bfloat16()
    b = (torch.randn(q3 + F, device="cuda", generator=g) * 0.1).bfloat16()
    ld = 4 * d + F
    out = torch.zeros(M, ld, device="cuda", dtype=torch.bfloat16)
    _gemm2(x, x2, _tile(w) if tiled else w, b, out, EPI_GELU, 2 if tiled else 1, nsplit=q3, ogap=d,
           N=q3 + F, K=d)
    ref_q = x.float() @ w[:q3].float().T + b[:q3].float()
    ref_f = _gelu(x2.float() @ w[q3:].float().T + b[q3:].float())
    tol = 2e-3 * (d / 256) ** 0.5
    assert (out[:, :q3].float() - ref_q).abs().max().item() <= tol + 2 ** -8 * ref_q.abs().max().item()
    assert (out[:, q3 + d:].float() - ref_f).abs().max().item() <= tol + 2 ** -8 * ref_f.abs().max().item()
    assert out[:, q3:q3 + d].abs().max().item() == 0      # the attention output's columns are untouched


@pytest.mark.parametrize("M", [1, 24, 64, 160, 256, 320, 448])
@pytest.mark.parametrize("V,d", [(50400, 4096), (50432, 6144), (50257, 768)])
def test_lm_head_fused_argmax(M, V, d):
    """K8 with the greedy argmax in the epilogue at the C2/C3/C4 LM heads:
    the packed (logit, lowest index) key equals torch's argmax of the fp32
    reference wherever its top-2 gap exceeds the accumulation error."""
    g = torch.Generator(device="cuda").manual_seed(M + V + d)
    x = (torch.randn(M, d, device="cuda", generator=g)).bfloat16()
    w = (torch.randn(V, d, device="cuda", generator=g) * 0.05).bfloat16()
    b = (torch.randn(V, device="cuda", generator=g) * 0.1).bfloat16()
    keys = torch.zeros(M, dtype=torch.int64, device="cuda")
    tiled = d % 64 == 0
    _gemm2(x, None, _tile(w) if tiled else w, b, None, 4, 2 if tiled else 1, keys=keys, N=V, K=d)
    ref = x.float() @ w.float().T + b.float()
    idx = 0xFFFFFFFF - (keys.cpu() & 0xFFFFFFFF)
    top2 = ref.topk(2, dim=1)
    gap = (top2.values[:, 0] - top2.values[:, 1]).cpu()
    sure = gap > 2e-2
    assert sure.sum() >= 0.8 * M
    assert torch.equal(idx[sure], top2.indices[:, 0].cpu()[sure])
    # near-ties: the chosen logit is within the error of the max
    picked = ref.gather(1, idx.cuda().long()[:, None])[:, 0]
    assert (top2.values[:, 0] - picked).abs().max().item() <= 2e-2
