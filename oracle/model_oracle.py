"""CPU model oracle for the fused decode step (test infrastructure only).

THIS IS A CHECKER, NOT PRODUCT CODE.  Only ``tests/``, ``__graft_entry__``
``smoke()`` and ``bench.py``'s CPU-baseline legs may import it.

Parity status: the reference (fusionsim) has NO model math -- SPEC.md:8,76
exclude weights, tensors and tokens -- so logits and token ids are
"parity unpinned by the reference".  This module states the block
definitions the framework adopted in plain numpy
fp32, following the paper's semantics:

  * PAPER.md:231   -- preprocessing passes the prompt once to build the
                      context (here: prompt tokens 0..P-2 enter the KV store)
  * an iteration is atomic: every fused request gains one
                      token, layer 0 through n-1, one shared pass
  * core.py:85     -- each request attends over its own step offset
  * SPEC.md:65, engine.py:81 -- stop lengths are pre-sampled, EOS ignored

Its KV store is keyed by REQUEST id, not by slot, so slot bookkeeping and
the device shuffle (K10) are checked implicitly: a wrong move corrupts the
device's context and its tokens/logits diverge from this oracle.

Families: gpt2 (sequential pre-LN, learned positions, tied head), gptj
(parallel residual, 1 LN, interleaved rotary), neox (parallel residual,
2 LNs, rotate-half rotary).  GELU = tanh approximation.
"""

from __future__ import annotations

import numpy as np

F32 = np.float32


def _ln(x, g, b, eps):
    mu = x.mean(axis=-1, keepdims=True, dtype=np.float64)
    var = ((x - mu) ** 2).mean(axis=-1, keepdims=True, dtype=np.float64)
    return ((x - mu) / np.sqrt(var + eps) * g + b).astype(F32)


def _gelu(x):
    return (0.5 * x * (1.0 + np.tanh(0.7978845608028654 * (x + 0.044715 * x ** 3)))).astype(F32)


def _rotary(v, pos, rot, family):
    """v: [H, hd] at one position."""
    if rot == 0:
        return v
    out = v.astype(np.float64).copy()
    j = np.arange(rot // 2)
    inv = 10000.0 ** (-2.0 * j / rot)
    ang = pos * inv
    c, s = np.cos(ang), np.sin(ang)
    if family == "gptj":
        a, b = v[:, 0:rot:2].astype(np.float64), v[:, 1:rot:2].astype(np.float64)
        out[:, 0:rot:2] = a * c - b * s
        out[:, 1:rot:2] = b * c + a * s
    else:
        h = rot // 2
        a, b = v[:, :h].astype(np.float64), v[:, h:rot].astype(np.float64)
        out[:, :h] = a * c - b * s
        out[:, h:rot] = b * c + a * s
    return out.astype(F32)


class GPTOracle:
    """Stateful decode oracle: ``step(rows)`` runs one fused iteration."""

    def __init__(self, family, n_layer, d_model, n_head, head_dim, d_ff, vocab, rotary_dim,
                 ln_eps, weights: dict, max_seq: int):
        self.family = family
        self.L, self.d, self.H, self.hd = n_layer, d_model, n_head, head_dim
        self.V, self.rot, self.eps, self.S = vocab, rotary_dim, ln_eps, max_seq
        self.w = {k: np.asarray(v, dtype=F32) for k, v in weights.items()}
        self.kv = {}          # rid -> [L, 2, S, H, hd]

    @classmethod
    def from_spec(cls, spec, weights, max_seq):
        return cls(spec.family, spec.n_layer, spec.d_model, spec.n_head, spec.head_dim, spec.d_ff,
                   spec.vocab, spec.rotary_dim, spec.ln_eps, weights, max_seq)

    def _lw(self, layer, key):
        return self.w.get(f"layers.{layer}.{key}")

    def _lin(self, x, w, b):
        y = x @ w.T
        return y + b if b is not None else y

    def _attention(self, layer, q, rows):
        out = np.empty((len(rows), self.H * self.hd), dtype=F32)
        scale = 1.0 / np.sqrt(self.hd)
        for i, (rid, pos, _) in enumerate(rows):
            K = self.kv[rid][layer, 0, :pos + 1]          # [ctx, H, hd]
            Vv = self.kv[rid][layer, 1, :pos + 1]
            qi = q[i].reshape(self.H, self.hd)
            s = np.einsum("hd,chd->hc", qi, K, dtype=np.float64) * scale
            s -= s.max(axis=1, keepdims=True)
            p = np.exp(s)
            p /= p.sum(axis=1, keepdims=True)
            out[i] = np.einsum("hc,chd->hd", p, Vv, dtype=np.float64).reshape(-1).astype(F32)
        return out

    def step(self, rows, want_logits=None):
        """rows: [(rid, pos, token)] of one fused iteration (prefill and
        decode rows alike).  Returns logits [n, V] for the rows whose index
        is in ``want_logits`` (all rows if None)."""
        for rid, pos, _ in rows:
            if rid not in self.kv:
                self.kv[rid] = np.zeros((self.L, 2, self.S, self.H, self.hd), dtype=F32)
        toks = np.array([t for _, _, t in rows])
        x = self.w["wte"][toks].astype(F32)
        if "wpe" in self.w:
            x = x + self.w["wpe"][np.array([p for _, p, _ in rows])]
        D = self.H * self.hd
        for layer in range(self.L):
            h = _ln(x, self._lw(layer, "ln1_g"), self._lw(layer, "ln1_b"), self.eps)
            h_mlp = h
            if self.family == "neox":
                h_mlp = _ln(x, self._lw(layer, "ln2_g"), self._lw(layer, "ln2_b"), self.eps)
            qkv = self._lin(h, self._lw(layer, "w_qkv"), self._lw(layer, "b_qkv"))
            q = np.empty((len(rows), D), dtype=F32)
            for i, (rid, pos, _) in enumerate(rows):
                qi = qkv[i, :D].reshape(self.H, self.hd)
                ki = qkv[i, D:2 * D].reshape(self.H, self.hd)
                vi = qkv[i, 2 * D:].reshape(self.H, self.hd)
                if self.family != "gpt2":
                    qi = _rotary(qi, pos, self.rot, self.family)
                    ki = _rotary(ki, pos, self.rot, self.family)
                q[i] = qi.reshape(-1)
                self.kv[rid][layer, 0, pos] = ki
                self.kv[rid][layer, 1, pos] = vi
            a = self._attention(layer, q, rows)
            x = x + self._lin(a, self._lw(layer, "w_o"), self._lw(layer, "b_o"))
            if self.family == "gpt2":
                h_mlp = _ln(x, self._lw(layer, "ln2_g"), self._lw(layer, "ln2_b"), self.eps)
            f = _gelu(self._lin(h_mlp, self._lw(layer, "w_fc"), self._lw(layer, "b_fc")))
            x = x + self._lin(f, self._lw(layer, "w_proj"), self._lw(layer, "b_proj"))
        idx = list(range(len(rows))) if want_logits is None else list(want_logits)
        if not idx:
            return np.zeros((0, self.V), dtype=F32)
        hf = _ln(x[idx], self.w["lnf_g"], self.w["lnf_b"], self.eps)
        wlm = self.w["w_lm"] if "w_lm" in self.w else self.w["wte"]
        logits = hf @ wlm.T
        if "b_lm" in self.w:
            logits = logits + self.w["b_lm"]
        return logits.astype(F32)

    def release(self, rid):
        self.kv.pop(rid, None)


def greedy(logits: np.ndarray) -> int:
    """max logit, lowest index on ties (matches the device argmax key)."""
    return int(np.argmax(logits))


def replay(oracle: GPTOracle, logits_log, prompts, gpu_tokens, stop=None):
    """Teacher-forced replay of a device run.

    logits_log: [(iteration, rids, kinds, device_logits[n_dec, V])] as
    recorded by CudaExecutor(capture_logits=True).  Inputs after the first
    decode step are the DEVICE's own tokens, so one ambiguous argmax cannot
    cascade.  Yields per decode row: (iteration, rid, step, oracle_logits,
    device_logits, device_token).
    """
    seen = {}
    for it, rids, kinds, dev in logits_log:
        rows = []
        want = []
        meta = []
        for i, (rid, kind) in enumerate(zip(rids, kinds)):
            if kind != 0:
                continue                      # orphan row: output discarded
            c = seen.get(rid, 0)
            P = len(prompts[rid])
            if c == 0:
                rows.extend((rid, j, prompts[rid][j]) for j in range(P - 1))
                tok = prompts[rid][P - 1]
            else:
                tok = gpu_tokens[rid][c - 1]
            want.append(len(rows))
            rows.append((rid, P - 1 + c, tok))
            meta.append((i, rid, c))
            seen[rid] = c + 1
        if not rows:
            continue
        lg = oracle.step(rows, want_logits=want)
        for k, (i, rid, c) in enumerate(meta):
            yield it, rid, c, lg[k], dev[i].numpy(), gpu_tokens[rid][c]
