"""Pin the model oracle's floating-point side to HF transformers (CPU).

The reference has no model math, so the block definitions in
oracle/model_oracle.py are this framework's documented choice.  This test
pins them to the public GPT-2, GPT-J and GPT-NeoX implementations of
``transformers`` (eager attention, fp32) on the reduced specs of each family:
the same seeded weights are loaded into the HF modules and the oracle's
logits over a full prompt (one fused step of prefill rows) must agree to
1e-4.  The fp32 torch restatement used at full shape (tests/torch_ref.py) is
checked against the oracle in the same test.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
transformers = pytest.importorskip("transformers")

from oracle.model_oracle import GPTOracle  # noqa: E402
from paper_2305_13484_b200.models import get_spec, init_weights  # noqa: E402
from torch_ref import _forward  # noqa: E402

T = 40


def _hf_gpt2(spec, w):
    cfg = transformers.GPT2Config(vocab_size=spec.vocab, n_positions=spec.max_pos, n_embd=spec.d_model,
                                  n_layer=spec.n_layer, n_head=spec.n_head, n_inner=spec.d_ff,
                                  activation_function="gelu_new", layer_norm_epsilon=spec.ln_eps,
                                  resid_pdrop=0.0, embd_pdrop=0.0, attn_pdrop=0.0,
                                  tie_word_embeddings=True, attn_implementation="eager")
    m = transformers.GPT2LMHeadModel(cfg).eval()
    sd = {"transformer.wte.weight": w["wte"], "transformer.wpe.weight": w["wpe"],
          "transformer.ln_f.weight": w["lnf_g"], "transformer.ln_f.bias": w["lnf_b"],
          "lm_head.weight": w["wte"]}
    for l in range(spec.n_layer):
        p, q = f"transformer.h.{l}.", f"layers.{l}."
        sd.update({p + "ln_1.weight": w[q + "ln1_g"], p + "ln_1.bias": w[q + "ln1_b"],
                   p + "ln_2.weight": w[q + "ln2_g"], p + "ln_2.bias": w[q + "ln2_b"],
                   p + "attn.c_attn.weight": w[q + "w_qkv"].t(), p + "attn.c_attn.bias": w[q + "b_qkv"],
                   p + "attn.c_proj.weight": w[q + "w_o"].t(), p + "attn.c_proj.bias": w[q + "b_o"],
                   p + "mlp.c_fc.weight": w[q + "w_fc"].t(), p + "mlp.c_fc.bias": w[q + "b_fc"],
                   p + "mlp.c_proj.weight": w[q + "w_proj"].t(), p + "mlp.c_proj.bias": w[q + "b_proj"]})
    return m, sd


def _hf_gptj(spec, w):
    cfg = transformers.GPTJConfig(vocab_size=spec.vocab, n_positions=2048, n_embd=spec.d_model,
                                  n_layer=spec.n_layer, n_head=spec.n_head, n_inner=spec.d_ff,
                                  rotary_dim=spec.rotary_dim, activation_function="gelu_new",
                                  layer_norm_epsilon=spec.ln_eps, resid_pdrop=0.0, embd_pdrop=0.0,
                                  attn_pdrop=0.0, tie_word_embeddings=False, attn_implementation="eager")
    m = transformers.GPTJForCausalLM(cfg).eval()
    D = spec.n_head * spec.head_dim
    sd = {"transformer.wte.weight": w["wte"], "transformer.ln_f.weight": w["lnf_g"],
          "transformer.ln_f.bias": w["lnf_b"], "lm_head.weight": w["w_lm"], "lm_head.bias": w["b_lm"]}
    for l in range(spec.n_layer):
        p, q = f"transformer.h.{l}.", f"layers.{l}."
        wq = w[q + "w_qkv"]
        sd.update({p + "ln_1.weight": w[q + "ln1_g"], p + "ln_1.bias": w[q + "ln1_b"],
                   p + "attn.q_proj.weight": wq[:D], p + "attn.k_proj.weight": wq[D:2 * D],
                   p + "attn.v_proj.weight": wq[2 * D:], p + "attn.out_proj.weight": w[q + "w_o"],
                   p + "mlp.fc_in.weight": w[q + "w_fc"], p + "mlp.fc_in.bias": w[q + "b_fc"],
                   p + "mlp.fc_out.weight": w[q + "w_proj"], p + "mlp.fc_out.bias": w[q + "b_proj"]})
    return m, sd


def _hf_neox(spec, w):
    H, hd = spec.n_head, spec.head_dim
    cfg = transformers.GPTNeoXConfig(vocab_size=spec.vocab, hidden_size=spec.d_model,
                                     num_hidden_layers=spec.n_layer, num_attention_heads=H,
                                     intermediate_size=spec.d_ff, hidden_act="gelu_new",
                                     max_position_embeddings=2048, layer_norm_eps=spec.ln_eps,
                                     use_parallel_residual=True, tie_word_embeddings=False,
                                     attention_dropout=0.0, hidden_dropout=0.0,
                                     rope_parameters={"rope_type": "default", "rope_theta": 10000.0,
                                                      "partial_rotary_factor": spec.rotary_dim / hd},
                                     attn_implementation="eager")
    m = transformers.GPTNeoXForCausalLM(cfg).eval()
    sd = {"gpt_neox.embed_in.weight": w["wte"], "gpt_neox.final_layer_norm.weight": w["lnf_g"],
          "gpt_neox.final_layer_norm.bias": w["lnf_b"], "embed_out.weight": w["w_lm"]}
    for l in range(spec.n_layer):
        p, q = f"gpt_neox.layers.{l}.", f"layers.{l}."
        # ours: rows [q heads | k heads | v heads]; HF: per head [q_h | k_h | v_h]
        wqkv = w[q + "w_qkv"].view(3, H, hd, -1).permute(1, 0, 2, 3).reshape(3 * H * hd, -1)
        bqkv = w[q + "b_qkv"].view(3, H, hd).permute(1, 0, 2).reshape(-1)
        sd.update({p + "input_layernorm.weight": w[q + "ln1_g"], p + "input_layernorm.bias": w[q + "ln1_b"],
                   p + "post_attention_layernorm.weight": w[q + "ln2_g"],
                   p + "post_attention_layernorm.bias": w[q + "ln2_b"],
                   p + "attention.query_key_value.weight": wqkv, p + "attention.query_key_value.bias": bqkv,
                   p + "attention.dense.weight": w[q + "w_o"], p + "attention.dense.bias": w[q + "b_o"],
                   p + "mlp.dense_h_to_4h.weight": w[q + "w_fc"], p + "mlp.dense_h_to_4h.bias": w[q + "b_fc"],
                   p + "mlp.dense_4h_to_h.weight": w[q + "w_proj"], p + "mlp.dense_4h_to_h.bias": w[q + "b_proj"]})
    return m, sd


BUILDERS = {"gpt2": _hf_gpt2, "gptj": _hf_gptj, "neox": _hf_neox}


@pytest.mark.parametrize("spec_name", ["tiny", "gpt2-mini", "gptj-mini", "neox-mini", "neox-mini-w"])
def test_oracle_matches_hf_transformers(spec_name):
    spec = get_spec(spec_name)
    w = init_weights(spec, seed=0, device="cpu", dtype=torch.float32)
    model, sd = BUILDERS[spec.family](spec, w)
    missing, unexpected = model.load_state_dict({k: v.contiguous() for k, v in sd.items()}, strict=False)
    # only non-persistent buffers (rotary caches, causal masks) may be left to the module
    assert not unexpected, unexpected
    assert all("rotary" in k or "bias" in k or "masked" in k for k in missing), missing
    g = np.random.default_rng(7)
    toks = [int(t) for t in g.integers(0, spec.vocab, T)]
    with torch.no_grad():
        hf = model(torch.tensor([toks])).logits[0].double().numpy()
    orc = GPTOracle.from_spec(spec, {k: v.numpy() for k, v in w.items()}, T)
    ours = orc.step([(0, p, t) for p, t in enumerate(toks)]).astype(np.float64)
    assert ours.shape == hf.shape
    err = float(np.abs(ours - hf).max())
    assert err <= 1e-4, (spec_name, err)
    # the full-shape reference (torch fp32, teacher-forced causal pass) is
    # the same math: it must equal the oracle too
    tr = _forward(spec, w, torch.tensor([toks]), 0)[0].double().numpy()
    assert float(np.abs(tr - ours).max()) <= 1e-4
