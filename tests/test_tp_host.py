"""Tensor-parallel host logic on CPU (no GPU here; the NCCL data path runs
inside fl_step on the box).

* Megatron shards reassemble into the full weights;
* a numpy simulation of the per-rank dataflow fl_step executes (head-local
  attention, row-parallel partial sums + all-reduce, vocab-parallel argmax
  with a packed max-reduce) equals the unsharded oracle;
* with world_size 2 over gloo, the NCCL unique id broadcast and the device
  clock agreement (max over ranks) keep the replicated schedule identical
  on every rank even when measured step times differ.
"""

import hashlib
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2305_13484_b200 as fl
from paper_2305_13484_b200.models import get_spec, init_weights, shard_tensor
from oracle.model_oracle import GPTOracle, _gelu, _ln, _rotary


@pytest.mark.parametrize("name,world", [("gptj-mini", 2), ("neox-mini", 2), ("neox-mini", 4),
                                        ("gpt2-mini", 2), ("gpt2-mini", 4)])
def test_shards_reassemble(name, world):
    spec = get_spec(name)
    full = init_weights(spec, seed=3)
    shards = [init_weights(spec, seed=3, rank=r, world=world) for r in range(world)]
    h, hd = spec.n_head, spec.head_dim
    for key, t in full.items():
        parts = [s[key] for s in shards]
        k = key.rsplit(".", 1)[-1]
        if k == "w_qkv":
            got = torch.cat([p.view(3, h // world, hd, -1) for p in parts], dim=1).reshape(t.shape)
        elif k == "b_qkv":
            got = torch.cat([p.view(3, h // world, hd) for p in parts], dim=1).reshape(-1)
        elif k in ("w_o", "w_proj"):
            got = torch.cat(parts, dim=1)
        elif k in ("w_fc", "b_fc", "w_lm", "b_lm"):
            got = torch.cat(parts, dim=0)
        else:
            assert all(torch.equal(p, t) for p in parts), key
            continue
        assert torch.equal(got, t), key
    vl = -(-spec.vocab // world)
    assert sum(s["w_lm"].shape[0] for s in shards) == spec.vocab
    assert all(s["w_lm"].shape[0] <= vl for s in shards)


def _tp_forward(spec, shards, rows, kv_store, merged=False):
    """numpy image of enqueue_step at tp = len(shards): returns the greedy
    token per row via the packed (logit, index) max-reduce.  merged: the
    parallel-residual path of fl_set_merged_out -- per rank [a | f] @
    [W_o | W_proj]^T, ONE all-reduce per layer, then + b_o + b_proj."""
    world = len(shards)
    w = [{k: v.numpy() for k, v in s.items()} for s in shards]
    hl, hd = spec.n_head // world, spec.head_dim
    D = hl * hd
    toks = np.array([t for _, _, t in rows])
    x = w[0]["wte"][toks].astype(np.float32)
    if "wpe" in w[0]:
        x = x + w[0]["wpe"][np.array([p for _, p, _ in rows])]
    for layer in range(spec.n_layer):
        g = lambda r, k: w[r].get(f"layers.{layer}.{k}")
        h = _ln(x, g(0, "ln1_g"), g(0, "ln1_b"), spec.ln_eps)
        h_mlp = _ln(x, g(0, "ln2_g"), g(0, "ln2_b"), spec.ln_eps) if spec.family == "neox" else h
        y = np.zeros_like(x)                       # all-reduce of attn-out partials
        a_rank = []
        for r in range(world):
            qkv = h @ g(r, "w_qkv").T + (g(r, "b_qkv") if g(r, "b_qkv") is not None else 0)
            a = np.zeros((len(rows), D), dtype=np.float32)
            for i, (rid, pos, _) in enumerate(rows):
                q = qkv[i, :D].reshape(hl, hd)
                k = qkv[i, D:2 * D].reshape(hl, hd)
                v = qkv[i, 2 * D:].reshape(hl, hd)
                if spec.family != "gpt2":
                    q, k = _rotary(q, pos, spec.rotary_dim, spec.family), _rotary(k, pos, spec.rotary_dim, spec.family)
                kv = kv_store.setdefault((rid, r, layer), {})
                kv[pos] = (k, v)
                K = np.stack([kv[p][0] for p in range(pos + 1)])
                V = np.stack([kv[p][1] for p in range(pos + 1)])
                s = np.einsum("hd,chd->hc", q, K) / np.sqrt(hd)
                p = np.exp(s - s.max(axis=1, keepdims=True))
                p /= p.sum(axis=1, keepdims=True)
                a[i] = np.einsum("hc,chd->hd", p, V).reshape(-1)
            a_rank.append(a)
            if not merged:
                y += a @ g(r, "w_o").T
        if merged:                                 # one all-reduce of [a|f] @ W_cat^T partials
            y = np.zeros_like(x)
            for r in range(world):
                f = _gelu(h_mlp @ g(r, "w_fc").T + g(r, "b_fc"))
                wcat = np.concatenate([g(r, "w_o"), g(r, "w_proj")], axis=1)
                y += np.concatenate([a_rank[r], f], axis=1) @ wcat.T
            bo = g(0, "b_o") if g(0, "b_o") is not None else 0
            x = x + y + bo + g(0, "b_proj")
            continue
        x = x + y + (g(0, "b_o") if g(0, "b_o") is not None else 0)
        if spec.family == "gpt2":
            h_mlp = _ln(x, g(0, "ln2_g"), g(0, "ln2_b"), spec.ln_eps)
        y = np.zeros_like(x)                       # all-reduce of FFN-down partials
        for r in range(world):
            f = _gelu(h_mlp @ g(r, "w_fc").T + g(r, "b_fc"))
            y += f @ g(r, "w_proj").T
        x = x + y + g(0, "b_proj")
    hf = _ln(x, w[0]["lnf_g"], w[0]["lnf_b"], spec.ln_eps)
    vl = -(-spec.vocab // world)
    best = [(-np.inf, 0)] * len(rows)
    for r in range(world):                         # packed max-reduce over ranks
        lg = hf @ w[r]["w_lm"].T + (w[r]["b_lm"] if "b_lm" in w[r] else 0)
        for i in range(len(rows)):
            j = int(np.argmax(lg[i]))
            cand = (float(lg[i, j]), -(r * vl + j))
            best[i] = max(best[i], cand)
    return [-b[1] for b in best], hf


@pytest.mark.parametrize("name,world", [("gptj-mini", 2), ("neox-mini", 4), ("gpt2-mini", 2)])
def test_tp_dataflow_matches_unsharded_oracle(name, world):
    spec = get_spec(name)
    full = init_weights(spec, seed=1)
    shards = [init_weights(spec, seed=1, rank=r, world=world) for r in range(world)]
    orc = GPTOracle.from_spec(spec, {k: v.numpy() for k, v in full.items()}, 64)
    prompt = [5, 17, 99, 3, 250, 7]
    rows = [(0, j, t) for j, t in enumerate(prompt)] + [(1, j, t) for j, t in enumerate(prompt[:3])]
    store = {}
    got, _ = _tp_forward(spec, shards, rows, store)
    want = orc.step(rows)
    assert got == [int(np.argmax(v)) for v in want]


@pytest.mark.parametrize("name,world", [("gptj-mini", 2), ("gptj-mini", 1), ("neox-mini", 4)])
def test_tp_merged_out_projection_matches_unsharded_oracle(name, world):
    """The merged out-projection dataflow (one all-reduce per layer) gives the
    oracle's tokens, as the two-all-reduce dataflow does."""
    spec = get_spec(name)
    full = init_weights(spec, seed=1)
    shards = [init_weights(spec, seed=1, rank=r, world=world) for r in range(world)]
    orc = GPTOracle.from_spec(spec, {k: v.numpy() for k, v in full.items()}, 64)
    prompt = [5, 17, 99, 3, 250, 7]
    rows = [(0, j, t) for j, t in enumerate(prompt)] + [(1, j, t) for j, t in enumerate(prompt[:3])]
    got, hf = _tp_forward(spec, shards, rows, {}, merged=True)
    want = orc.step(rows)
    assert got == [int(np.argmax(v)) for v in want]
    _, hf2 = _tp_forward(spec, shards, rows, {}, merged=False)
    assert np.abs(hf - hf2).max() < 1e-3


# ---------------------------------------------------------------- gloo, world 2
def _worker(rank, world, port, out):
    """One TP rank driving the REAL executor host path (CudaExecutor on a
    stub library, tests/stub_device.py): weight sharding, comm-id broadcast
    and fl_comm_init, per-step row tables, shuffles, and the device clock
    agreed across ranks by max_reduce_clock -- with rank-dependent step
    times, the replicated schedules must stay identical."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from stub_device import stub_device
        from paper_2305_13484_b200.executor import CudaExecutor
        from paper_2305_13484_b200.models import get_spec
        from paper_2305_13484_b200.tp import make_comm_id, max_reduce_clock
        cid = make_comm_id(rank, device=torch.device("cpu"), id_fn=lambda: bytes(range(128)))
        sc = fl.Scenario("tp", fl.Discipline.FUSION, 24, fl.PoissonArrival(3.0),
                         fl.UniformLength(2, 20), 20, input_len=8)
        reqs = fl.build_requests(sc, 7)
        spec = get_spec("gptj-mini")
        prompts = fl.synthetic_prompts(reqs, spec.vocab, 7)
        with stub_device(rank) as rec:
            ex = CudaExecutor(spec, prompts, dtype="bf16", pool_slots=24, input_len=8, max_new_tokens=20,
                              state_slots=64, tp_rank=rank, tp_size=world, comm_id=cid, device="cpu")
            ex.clock_reduce = max_reduce_clock(device=torch.device("cpu"))
            st = fl.FusionStream(reqs, fl.CostParams(preprocess_ms=0.0), fl.TPConfig(world),
                                 executor=ex, clock="device")
            fl.drive(st)
            hl = (ex.mdesc.tp_rank, ex.mdesc.tp_size, int(ex.kv.shape[3]))
        digest = hashlib.sha256("\n".join(fl.Trace("f", st.events).format_lines()).encode()).hexdigest()
        steps = hashlib.sha256(repr(rec.steps).encode()).hexdigest()
        out.put((rank, rec.comm, digest, st.iteration_index, steps, len(rec.shuffles), ex.tp_layout, hl))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_comm_id_and_clock_agreement():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=180) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, c0, d0, n0, s0, sh0, lay0, hl0), (r1, c1, d1, n1, s1, sh1, lay1, hl1) = res
    # the NCCL unique id reached both ranks, each initialised its own rank of 2
    assert c0 == (bytes(range(128)), 0, 2) and c1 == (bytes(range(128)), 1, 2)
    # replicated schedule: identical traces, row tables and shuffles per step
    assert d0 == d1 and n0 == n1 > 0
    assert s0 == s1 and sh0 == sh1 > 0
    # under TP the north star's layout: an all-reduce after attn-out AND FFN-down
    assert lay0 == lay1 == "two all-reduces per layer (after attn-out and after FFN-down)"
    # each rank holds its own half of the heads in its KV pool
    assert hl0 == (0, 2, 1) and hl1 == (1, 2, 1)
