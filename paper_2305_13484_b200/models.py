"""Model shapes of the benchmark configs and seeded weights.

The reference carries no model at all; block definitions are this
framework's documented choice:

* gpt2  -- sequential pre-LN blocks, learned positions, tied LM head (C1, C2)
* gptj  -- parallel residual, one LN, interleaved rotary on the first
           ``rotary_dim`` dims of each head, LM head with bias (C3, C5)
* neox  -- parallel residual, two LNs, rotate-half rotary (C4)

GELU is the tanh approximation; attention scale 1/sqrt(head_dim).

Weights are synthetic (no checkpoints exist offline): N(0, 0.02) for linear
and embedding matrices and biases, LN gamma = 1 + N(0, 0.02), beta =
N(0, 0.02); the untied LM heads use std ``lm_std`` so greedy margins clear
the bf16 tolerance.  Every tensor is drawn from its own seeded generator
(seed, tensor index), so a tensor is reproducible in isolation.
"""

from __future__ import annotations

from dataclasses import dataclass, replace

import torch

LAYER_KEYS = ("ln1_g", "ln1_b", "ln2_g", "ln2_b", "w_qkv", "b_qkv", "w_o", "b_o",
              "w_fc", "b_fc", "w_proj", "b_proj")


@dataclass(frozen=True)
class ModelSpec:
    name: str
    family: str          # gpt2 | gptj | neox
    n_layer: int
    d_model: int
    n_head: int
    head_dim: int
    d_ff: int
    vocab: int
    max_pos: int = 2048
    rotary_dim: int = 0
    ln_eps: float = 1e-5
    lm_std: float = 0.02

    @property
    def tied(self) -> bool:
        return self.family == "gpt2"

    def kv_bytes_per_token(self, dtype_bytes: int, tp: int = 1) -> int:
        return 2 * self.n_layer * (self.n_head // tp) * self.head_dim * dtype_bytes

    def n_params(self) -> int:
        d, f, v = self.d_model, self.d_ff, self.vocab
        per = 4 * d * d + 2 * d * f
        return self.n_layer * per + v * d * (1 if self.tied else 2)


SPECS = {
    # C1: tiny GPT (builder's choice of V and F)
    "tiny": ModelSpec("tiny", "gpt2", 4, 256, 4, 64, 1024, 1024, max_pos=256),
    # C2: GPT-2 small
    "gpt2-small": ModelSpec("gpt2-small", "gpt2", 12, 768, 12, 64, 3072, 50257, max_pos=1024),
    # C3 / C5: GPT-J 6B
    "gptj-6b": ModelSpec("gptj-6b", "gptj", 28, 4096, 16, 256, 16384, 50400, rotary_dim=64,
                         lm_std=0.05),
    # C4: GPT-NeoX 20B
    "neox-20b": ModelSpec("neox-20b", "neox", 44, 6144, 64, 96, 24576, 50432, rotary_dim=24,
                          lm_std=0.05),
    # reduced shapes of the same families for parity tests
    "gptj-mini": ModelSpec("gptj-mini", "gptj", 2, 512, 2, 256, 1024, 2048, rotary_dim=64,
                           lm_std=0.05),
    "neox-mini": ModelSpec("neox-mini", "neox", 2, 384, 4, 96, 768, 2048, rotary_dim=24,
                           lm_std=0.05),
    # 3 * d_model a multiple of 256: exercises the merged QKV / FFN-up GEMM
    "neox-mini-w": ModelSpec("neox-mini-w", "neox", 2, 768, 8, 96, 1536, 2048, rotary_dim=24,
                             lm_std=0.05),
    "gpt2-mini": ModelSpec("gpt2-mini", "gpt2", 2, 256, 4, 64, 1024, 4096, max_pos=1024),
}


def get_spec(name: str, **overrides) -> ModelSpec:
    spec = SPECS[name]
    return replace(spec, **overrides) if overrides else spec


def _shapes(spec: ModelSpec) -> list:
    d, f, hd, h = spec.d_model, spec.d_ff, spec.head_dim, spec.n_head
    qkv = 3 * h * hd
    out = [("wte", (spec.vocab, d), "w")]
    if spec.family == "gpt2":
        out.append(("wpe", (spec.max_pos, d), "w"))
    for layer in range(spec.n_layer):
        p = f"layers.{layer}."
        out += [(p + "ln1_g", (d,), "g"), (p + "ln1_b", (d,), "b")]
        if spec.family != "gptj":
            out += [(p + "ln2_g", (d,), "g"), (p + "ln2_b", (d,), "b")]
        out += [(p + "w_qkv", (qkv, d), "w")]
        if spec.family != "gptj":
            out += [(p + "b_qkv", (qkv,), "b")]
        out += [(p + "w_o", (d, h * hd), "w")]
        if spec.family != "gptj":
            out += [(p + "b_o", (d,), "b")]
        out += [(p + "w_fc", (f, d), "w"), (p + "b_fc", (f,), "b"),
                (p + "w_proj", (d, f), "w"), (p + "b_proj", (d,), "b")]
    out += [("lnf_g", (d,), "g"), ("lnf_b", (d,), "b")]
    if not spec.tied:
        out.append(("w_lm", (spec.vocab, d), "lm"))
        if spec.family == "gptj":
            out.append(("b_lm", (spec.vocab,), "b"))
    return out


def _draw(spec: ModelSpec, idx: int, shape, kind: str, seed: int, dev) -> torch.Tensor:
    g = torch.Generator(device=dev)
    g.manual_seed((seed * 1_000_003 + idx * 7_919) & 0x7FFFFFFFFFFFFFFF)
    t = torch.randn(shape, generator=g, device=dev, dtype=torch.float32)
    if kind == "g":
        return t.mul_(0.02).add_(1.0)
    return t.mul_(spec.lm_std if kind == "lm" else 0.02)


def shard_tensor(spec: ModelSpec, name: str, t: torch.Tensor, rank: int, world: int) -> torch.Tensor:
    """Megatron slicing of one full tensor: q/k/v heads and FFN columns
    column-parallel, attn-out and FFN-down row-parallel, vocab-parallel LM
    head (ceil(V/world) rows per rank); everything else replicated."""
    if world == 1:
        return t
    key = name.rsplit(".", 1)[-1]
    h, hd = spec.n_head, spec.head_dim
    hl, fl = h // world, spec.d_ff // world
    if key == "w_qkv":
        return t.view(3, h, hd, -1)[:, rank * hl:(rank + 1) * hl].reshape(3 * hl * hd, -1).contiguous()
    if key == "b_qkv":
        return t.view(3, h, hd)[:, rank * hl:(rank + 1) * hl].reshape(-1).contiguous()
    if key == "w_o":
        return t[:, rank * hl * hd:(rank + 1) * hl * hd].contiguous()
    if key in ("w_fc", "b_fc"):
        return t[rank * fl:(rank + 1) * fl].contiguous()
    if key == "w_proj":
        return t[:, rank * fl:(rank + 1) * fl].contiguous()
    if key in ("w_lm", "b_lm"):
        vl = (spec.vocab + world - 1) // world
        return t[rank * vl:min(spec.vocab, (rank + 1) * vl)].contiguous()
    return t


def init_weights(spec: ModelSpec, seed: int = 0, device="cpu", dtype=torch.float32,
                 rank: int = 0, world: int = 1) -> dict:
    """This rank's weights.  Each full tensor is drawn in fp32 from its own
    seeded generator, sliced for (rank, world) and rounded once to ``dtype``,
    so every rank holds a shard of the same model.  ``w_lm`` is always
    present (for tied models it is the vocab slice of ``wte``)."""
    out = {}
    dev = torch.device(device)
    for idx, (name, shape, kind) in enumerate(_shapes(spec)):
        t = _draw(spec, idx, shape, kind, seed, dev)
        out[name] = shard_tensor(spec, name, t, rank, world).to(dtype)
        del t
    if spec.tied:
        out["w_lm"] = shard_tensor(spec, "w_lm", out["wte"], rank, world)
    return out
