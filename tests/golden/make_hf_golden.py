"""Pin oracle/model_ref.py against transformers' Mixtral / Mistral (third-party,
not vendored in /root/reference; SURVEY.md §8c "Third-party arithmetic").

    python tests/golden/make_hf_golden.py     → tests/golden/hf_tiny.npz

Loads the tiny pair's deterministic weights (oracle/tiny.py) into
MixtralForCausalLM / MistralForCausalLM (fp32, eager attention) and records
full-sequence logits for two prompts, plus the routing of layer 0.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
from oracle import tiny  # noqa: E402
from transformers import MistralConfig, MistralForCausalLM, MixtralConfig, MixtralForCausalLM  # noqa: E402


def hf_state(arch, W, moe):
    sd = {"model.embed_tokens.weight": W["embed"], "model.norm.weight": W["final_norm"], "lm_head.weight": W["lm_head"]}
    for i, L in enumerate(W["layers"]):
        p = f"model.layers.{i}."
        sd[p + "input_layernorm.weight"] = L["attn_norm"]
        sd[p + "post_attention_layernorm.weight"] = L["ffn_norm"]
        for n in ("q", "k", "v", "o"):
            sd[p + f"self_attn.{n}_proj.weight"] = L["w" + n]
        if moe:
            sd[p + "mlp.gate.weight"] = L["router"]
            sd[p + "mlp.experts.gate_up_proj"] = np.concatenate([L["w_gate"], L["w_up"]], axis=1)
            sd[p + "mlp.experts.down_proj"] = L["w_down"]
        else:
            sd[p + "mlp.gate_proj.weight"] = L["w_gate"]
            sd[p + "mlp.up_proj.weight"] = L["w_up"]
            sd[p + "mlp.down_proj.weight"] = L["w_down"]
    return {k: torch.from_numpy(np.ascontiguousarray(v, np.float32)) for k, v in sd.items()}


def main():
    tw, dw = tiny.weights()
    t, d = tiny.TARGET, tiny.DRAFT
    common = dict(rope_theta=t.rope_theta, rms_norm_eps=t.eps, tie_word_embeddings=False,
                  max_position_embeddings=4096, attn_implementation="eager")
    tc = MixtralConfig(vocab_size=t.vocab, hidden_size=t.hidden, intermediate_size=t.inter,
                       num_hidden_layers=t.n_layer, num_attention_heads=t.n_head, num_key_value_heads=t.n_kv_head,
                       head_dim=t.head_dim, num_local_experts=t.n_expert, num_experts_per_tok=t.top_k, **common)
    dc = MistralConfig(vocab_size=d.vocab, hidden_size=d.hidden, intermediate_size=d.inter,
                       num_hidden_layers=d.n_layer, num_attention_heads=d.n_head, num_key_value_heads=d.n_kv_head,
                       head_dim=d.head_dim, **common)
    tm = MixtralForCausalLM(tc).eval()
    dm = MistralForCausalLM(dc).eval()
    tm.load_state_dict(hf_state(t, tw, True), strict=True)
    dm.load_state_dict(hf_state(d, dw, False), strict=True)
    prompts = tiny.prompts(2, seed=99, lo=10, hi=20)
    out = {}
    with torch.no_grad():
        for i, p in enumerate(prompts):
            ids = torch.from_numpy(p.astype(np.int64))[None]
            out[f"prompt{i}"] = p
            out[f"target_logits{i}"] = tm(ids).logits[0].float().numpy()
            out[f"draft_logits{i}"] = dm(ids).logits[0].float().numpy()
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "hf_tiny.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, {k: v.shape for k, v in out.items()})


if __name__ == "__main__":
    main()
