"""fp32 torch reference of the model math, for full-shape parity (test-only).

The numpy oracle (oracle/model_oracle.py) replays a device run iteration by
iteration and is the pinned statement of the block definitions (tests/
test_oracle_hf.py pins it to HF transformers).  At the benchmarked shapes
(GPT-J 6B, NeoX 20B, GPT-2 small with 100+ requests) a CPU replay would take
hours, so this module restates the SAME math in plain torch fp32 on the GPU
and evaluates it per request over the full teacher-forced sequence in one
causal pass:

    tokens = prompt[0..P-1] + device_tokens[0..stop-2]
    logits at position P-1+c  ->  must predict device_tokens[c]

Because every request's stream depends only on its own tokens (PAPER.md
234-236: the fused iteration is atomic and rows are independent), the value
at (rid, c) equals the oracle's value at the iteration that produced it, so
batching, slot maps and shuffles of the device run are checked implicitly --
exactly like the rid-keyed numpy oracle.

Weights are the caller's (bf16 or fp32) tensors, upcast layer by layer to
fp32 (true fp32 matmuls: TF32 is switched off while this runs).
"""

from __future__ import annotations

import math

import torch


def _ln(x, g, b, eps):
    mu = x.mean(-1, keepdim=True)
    var = (x - mu).pow(2).mean(-1, keepdim=True)
    return (x - mu) * torch.rsqrt(var + eps) * g.float() + b.float()


def _gelu(x):
    return 0.5 * x * (1.0 + torch.tanh(0.7978845608028654 * (x + 0.044715 * x ** 3)))


def _rotary(v, pos, rot, family):
    """v: [B, T, H, hd]; pos: [T] absolute positions (oracle _rotary)."""
    if rot == 0:
        return v
    j = torch.arange(rot // 2, device=v.device, dtype=torch.float64)
    inv = 10000.0 ** (-2.0 * j / rot)
    ang = pos.double()[:, None] * inv[None, :]                   # [T, rot/2]
    c = torch.cos(ang).float()[None, :, None, :]
    s = torch.sin(ang).float()[None, :, None, :]
    out = v.clone()
    if family == "gptj":
        a, b = v[..., 0:rot:2], v[..., 1:rot:2]
        out[..., 0:rot:2] = a * c - b * s
        out[..., 1:rot:2] = b * c + a * s
    else:
        h = rot // 2
        a, b = v[..., :h], v[..., h:rot]
        out[..., :h] = a * c - b * s
        out[..., h:rot] = b * c + a * s
    return out


@torch.no_grad()
def forward_logits(spec, weights: dict, tokens: torch.Tensor, first: int) -> torch.Tensor:
    """tokens: [B, T] int64 on the GPU (right-padded; padding only affects
    positions after it under the causal mask).  Returns fp32 logits
    [B, T - first, V] for positions first..T-1."""
    tf32 = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        return _forward(spec, weights, tokens, first)
    finally:
        torch.backends.cuda.matmul.allow_tf32 = tf32


def _w(weights, key):
    t = weights.get(key)
    return None if t is None else t.float()


def _lin(x, w, b):
    y = x @ w.t()
    return y + b if b is not None else y


def _forward(spec, weights, tokens, first):
    B, T = tokens.shape
    H, hd, d = spec.n_head, spec.head_dim, spec.d_model
    D = H * hd
    dev = tokens.device
    pos = torch.arange(T, device=dev)
    x = weights["wte"][tokens].float()
    if spec.family == "gpt2":
        x = x + weights["wpe"][pos].float()[None]
    mask = torch.ones(T, T, dtype=torch.bool, device=dev).tril()
    scale = 1.0 / math.sqrt(hd)
    for l in range(spec.n_layer):
        p = f"layers.{l}."
        h = _ln(x, weights[p + "ln1_g"], weights[p + "ln1_b"], spec.ln_eps)
        h_mlp = h
        if spec.family == "neox":
            h_mlp = _ln(x, weights[p + "ln2_g"], weights[p + "ln2_b"], spec.ln_eps)
        qkv = _lin(h, _w(weights, p + "w_qkv"), _w(weights, p + "b_qkv"))
        q = qkv[..., :D].view(B, T, H, hd)
        k = qkv[..., D:2 * D].view(B, T, H, hd)
        v = qkv[..., 2 * D:].view(B, T, H, hd)
        if spec.family != "gpt2":
            q = _rotary(q, pos, spec.rotary_dim, spec.family)
            k = _rotary(k, pos, spec.rotary_dim, spec.family)
        s = torch.einsum("bthd,bshd->bhts", q, k) * scale
        s = s.masked_fill(~mask, float("-inf"))
        a = torch.einsum("bhts,bshd->bthd", torch.softmax(s, dim=-1), v).reshape(B, T, D)
        del s, q, k, v, qkv
        x = x + _lin(a, _w(weights, p + "w_o"), _w(weights, p + "b_o"))
        if spec.family == "gpt2":
            h_mlp = _ln(x, weights[p + "ln2_g"], weights[p + "ln2_b"], spec.ln_eps)
        f = _gelu(_lin(h_mlp, _w(weights, p + "w_fc"), _w(weights, p + "b_fc")))
        x = x + _lin(f, _w(weights, p + "w_proj"), _w(weights, p + "b_proj"))
    hf = _ln(x[:, first:], weights["lnf_g"], weights["lnf_b"], spec.ln_eps)
    wlm = weights["w_lm"] if "w_lm" in weights else weights["wte"]
    logits = hf @ wlm.float().t()
    if "b_lm" in weights:
        logits = logits + weights["b_lm"].float()
    return logits


def check_run(spec, weights, ex, prompts, *, atol, rtol, margin, batch_tokens=16384):
    """Compare a device run (CudaExecutor with capture_logits=True) with the
    fp32 reference.  Returns stats: rows checked, exact / ambiguous /
    mismatched greedy tokens, worst |Δlogit| - rtol*|ref| (must be <= atol),
    and the max |Δlogit| seen."""
    toks = ex.tokens()
    # (rid, c) -> device logits, in the order the device produced them
    dev_logits = {}
    seen = {}
    for _, rids, kinds, lg in ex.logits_log:
        for i, (rid, kind) in enumerate(zip(rids, kinds)):
            if kind != 0:
                continue
            c = seen.get(rid, 0)
            seen[rid] = c + 1
            dev_logits[(rid, c)] = lg[i]
    stats = {"rows": 0, "exact": 0, "ambiguous": 0, "mismatched": 0, "worst_excess": -1e30,
             "max_abs": 0.0, "requests": 0}
    rids = sorted(seen)
    P = {rid: len(prompts[rid]) for rid in rids}
    # group requests of equal prompt length; batch by token budget
    groups = {}
    for rid in rids:
        groups.setdefault(P[rid], []).append(rid)
    for plen, members in groups.items():
        members.sort(key=lambda r: -seen[r])
        i = 0
        while i < len(members):
            T = plen - 1 + seen[members[i]]
            nb = max(1, batch_tokens // T)
            chunk = members[i:i + nb]
            i += nb
            seqs = torch.zeros(len(chunk), T, dtype=torch.long)
            for b, rid in enumerate(chunk):
                s = list(prompts[rid]) + list(toks[rid][:seen[rid] - 1])
                seqs[b, :len(s)] = torch.tensor(s)
            ref = forward_logits(spec, weights, seqs.cuda(), plen - 1)    # [b, T-P+1, V]
            for b, rid in enumerate(chunk):
                stats["requests"] += 1
                n = seen[rid]
                lo = ref[b, :n]
                ld = torch.stack([dev_logits[(rid, c)] for c in range(n)]).to(lo.device)[:, :spec.vocab]
                diff = (lo - ld).abs()
                stats["max_abs"] = max(stats["max_abs"], float(diff.max()))
                stats["worst_excess"] = max(stats["worst_excess"], float((diff - rtol * lo.abs()).max()))
                dt = torch.tensor(toks[rid][:n], device=lo.device)
                top = lo.argmax(-1)
                top2 = lo.topk(2, dim=-1).values
                gap = top2[:, 0] - top2[:, 1]
                at_tok = lo.gather(1, dt[:, None])[:, 0]
                exact = dt == top
                amb = ~exact & ((gap < margin) | (at_tok >= top2[:, 0] - margin))
                stats["rows"] += n
                stats["exact"] += int(exact.sum())
                stats["ambiguous"] += int(amb.sum())
                stats["mismatched"] += int((~exact & ~amb).sum())
            del ref
    return stats
