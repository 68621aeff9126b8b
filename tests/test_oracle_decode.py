"""Pin for oracle c4 (decode step): token-by-token decode over the KV cache
equals a one-shot causal forward of the HF transformers reference models
(textbook equivalence; independent library implementation) in float64 on the
same weights. CPU only."""
import numpy as np
import pytest
import torch

from oracle.decode import Decoder
from synth import models, weights, workload

transformers = pytest.importorskip("transformers")


def hf_opt(m, layers, glob):
    from transformers import OPTConfig, OPTForCausalLM
    cfg = OPTConfig(vocab_size=m.vocab, hidden_size=m.d_model, num_hidden_layers=m.n_layers,
                    ffn_dim=m.ffn_dim, num_attention_heads=m.n_heads,
                    max_position_embeddings=m.max_pos, do_layer_norm_before=True,
                    word_embed_proj_dim=m.d_model, enable_bias=True, dropout=0.0,
                    activation_function="relu", layer_norm_elementwise_affine=True)
    model = OPTForCausalLM(cfg).double().eval()
    d = m.d_model
    sd = {}
    p = "model.decoder."
    sd[p + "embed_tokens.weight"] = glob["embed"]
    sd[p + "embed_positions.weight"] = glob["pos_embed"]
    sd[p + "final_layer_norm.weight"] = glob["lnf_g"]
    sd[p + "final_layer_norm.bias"] = glob["lnf_b"]
    sd["lm_head.weight"] = glob["embed"]
    for i, W in enumerate(layers):
        q = f"{p}layers.{i}."
        for j, nm in enumerate(("q_proj", "k_proj", "v_proj")):
            sd[q + f"self_attn.{nm}.weight"] = W["w_qkv"][j * d:(j + 1) * d]
            sd[q + f"self_attn.{nm}.bias"] = W["b_qkv"][j * d:(j + 1) * d]
        sd[q + "self_attn.out_proj.weight"] = W["w_o"]
        sd[q + "self_attn.out_proj.bias"] = W["b_o"]
        sd[q + "self_attn_layer_norm.weight"] = W["ln1_g"]
        sd[q + "self_attn_layer_norm.bias"] = W["ln1_b"]
        sd[q + "final_layer_norm.weight"] = W["ln2_g"]
        sd[q + "final_layer_norm.bias"] = W["ln2_b"]
        sd[q + "fc1.weight"] = W["w_fc1"]
        sd[q + "fc1.bias"] = W["b_fc1"]
        sd[q + "fc2.weight"] = W["w_fc2"]
        sd[q + "fc2.bias"] = W["b_fc2"]
    sd = {k: v.double() for k, v in sd.items()}
    missing, unexpected = model.load_state_dict(sd, strict=False)
    assert not unexpected, unexpected
    assert all("lm_head" in k for k in missing), missing
    return model


def hf_llama(m, layers, glob):
    from transformers import LlamaConfig, LlamaForCausalLM
    cfg = LlamaConfig(vocab_size=m.vocab, hidden_size=m.d_model, intermediate_size=m.ffn_dim,
                      num_hidden_layers=m.n_layers, num_attention_heads=m.n_heads,
                      num_key_value_heads=m.n_kv_heads, head_dim=m.head_dim,
                      max_position_embeddings=m.max_pos, rms_norm_eps=m.norm_eps,
                      rope_theta=m.rope_theta, tie_word_embeddings=False,
                      attention_bias=False, mlp_bias=False)
    model = LlamaForCausalLM(cfg).double().eval()
    H, Hk, D, f = m.n_heads, m.n_kv_heads, m.head_dim, m.ffn_dim
    sd = {"model.embed_tokens.weight": glob["embed"], "model.norm.weight": glob["normf_g"],
          "lm_head.weight": glob["lm_head"]}
    for i, W in enumerate(layers):
        q = f"model.layers.{i}."
        sd[q + "self_attn.q_proj.weight"] = W["w_qkv"][: H * D]
        sd[q + "self_attn.k_proj.weight"] = W["w_qkv"][H * D:(H + Hk) * D]
        sd[q + "self_attn.v_proj.weight"] = W["w_qkv"][(H + Hk) * D:]
        sd[q + "self_attn.o_proj.weight"] = W["w_o"]
        sd[q + "mlp.gate_proj.weight"] = W["w_gateup"][:f]
        sd[q + "mlp.up_proj.weight"] = W["w_gateup"][f:]
        sd[q + "mlp.down_proj.weight"] = W["w_down"]
        sd[q + "input_layernorm.weight"] = W["rms1_g"]
        sd[q + "post_attention_layernorm.weight"] = W["rms2_g"]
    sd = {k: v.double() for k, v in sd.items()}
    missing, unexpected = model.load_state_dict(sd, strict=False)
    assert not unexpected and not missing, (missing, unexpected)
    return model


@pytest.mark.parametrize("shape", [models.TOY, models.TOY_LLAMA])
def test_decode_equals_hf_causal_forward(shape):
    m = shape
    layers = [weights.layer_tensors(m, l, seed=11) for l in range(m.n_layers)]
    glob = weights.global_tensors(m, seed=11)
    T = 24
    seqs = [0, 1]
    toks = np.array([[workload.teacher_tokens(s, t, m.vocab) for t in range(T)] for s in seqs])
    model = (hf_opt if m.family == models.OPT else hf_llama)(m, layers, glob)
    with torch.no_grad():
        out = model(torch.from_numpy(toks), output_hidden_states=True)
    ref_logits = out.logits.numpy()
    dec = Decoder(m, layers, glob, round_points=False)
    for t in range(T):
        hid, logits, am = dec.step(seqs, toks[:, t], [t, t])
        np.testing.assert_allclose(logits, ref_logits[:, t], rtol=1e-6, atol=1e-6 * np.abs(ref_logits).max())
        if m.family == models.OPT:
            np.testing.assert_allclose(hid, out.hidden_states[-1][:, t].numpy(), rtol=1e-6, atol=1e-9)


def test_rounding_points_are_small_perturbation():
    m = models.TOY
    layers = [weights.layer_tensors(m, l, seed=2) for l in range(m.n_layers)]
    glob = weights.global_tensors(m, seed=2)
    a, b = Decoder(m, layers, glob, True), Decoder(m, layers, glob, False)
    for t in range(8):
        ha, _, _ = a.step([0], [t * 3], [t])
        hb, _, _ = b.step([0], [t * 3], [t])
    rel = np.sqrt(((ha - hb) ** 2).mean() / (hb ** 2).mean())
    assert 0 < rel < 2e-2


@pytest.mark.parametrize("shape", [models.TOY, models.TOY_LLAMA])
def test_noise_model_bound_covers_real_bf16_rounding(shape):
    """The end-to-end tolerance is derived from the first-order bf16 noise model
    (tests/c4_bounds.py). Check the model against real round-to-nearest-even bf16
    at the same points (the rounded twin): the derived bound must cover it, and
    sigma -> 0 must reproduce the exact decoder bit for bit."""
    import c4_bounds as CB
    layers = [weights.layer_tensors(shape, l, seed=4) for l in range(shape.n_layers)]
    glob = weights.global_tensors(shape, seed=4)
    B, steps = 4, 12

    def script(dec):
        out = []
        for t in range(steps):
            h, lg, _ = dec.step(list(range(B)), [workload.teacher_tokens(s, t, shape.vocab) for s in range(B)],
                                [t] * B)
            out.append((h, lg))
        return out
    exact, bounds = CB.predict(shape, layers, glob, script)
    rounded = script(Decoder(shape, layers, glob, round_points=True))
    for t in range(steps):
        rel, mx = CB.check(rounded[t][0], exact[t][0], bounds[t], t)
        assert rel > 0
    zero = script(Decoder(shape, layers, glob, noise=(0.0, np.random.default_rng(0), "survey")))
    for t in range(steps):
        assert np.array_equal(zero[t][0], exact[t][0])
    # an all-bf16 implementation (every SURVEY c4 point) is predicted to be noisier
    _, b_survey = CB.predict(shape, layers, glob, script, draws=2, points="survey")
    assert b_survey[-1][0] > bounds[-1][0]
    # argmax decidability is sound: where decidable, the rounded twin's argmax is the exact one
    E = CB.lm_head(shape, glob)
    for t in range(steps):
        ok = CB.argmax_decidable(E, rounded[t][0], exact[t][0], exact[t][1])
        for s in range(B):
            if ok[s]:
                assert np.argmax(E @ rounded[t][0][s]) == np.argmax(exact[t][1][s])
