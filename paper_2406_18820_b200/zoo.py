"""Model specs used as reshard workloads.

``make_model`` mirrors the reference model zoo (ucp/models.py:126-222):
DenseGPT, MoE (fused experts, one Shard-NC segment per expert) and GQA (fused
QKV with unequal q/k/v segments). ``llama_spec`` encodes LLaMA-2 7B/13B/70B
exactly as SURVEY §8(d) prescribes (fused QKV and fused gate/up as Shard-NC,
RMSNorm as replicated LAYERNORM_WEIGHT, untied head); the element totals
equal the published LLaMA-2 parameter counts.

``BENCH_CONFIGS`` are the five BASELINE.json workloads as (spec, src, tgt).
"""

from __future__ import annotations

from ._errors import ModelConfigError
from .spec import ModelSpec, ParallelConfig, ParamKind, ParamSpec, ZeroStage

VOCAB = 512
MAX_TP = 8
FAMILIES = ("DenseGPT", "MoE", "GQA")

K = ParamKind


def make_model(family: str, scale: dict) -> ModelSpec:
    """ModelSpec for a reference family at a scale (ucp/models.py:126-222)."""
    if family not in FAMILIES:
        raise ModelConfigError(f"unknown family {family!r}; expected one of {FAMILIES}")
    try:
        n_layers, hidden = int(scale["n_layers"]), int(scale["hidden"])
    except KeyError as e:
        raise ModelConfigError(f"scale missing key {e}") from e
    if n_layers < 0:
        raise ModelConfigError("n_layers must be >= 0")
    if hidden <= 0 or hidden % (2 * MAX_TP):
        raise ModelConfigError(f"hidden must be a positive multiple of {2 * MAX_TP}")
    n_exp = int(scale.get("n_experts", 0))
    qh, kvh = int(scale.get("q_heads", 0)), int(scale.get("kv_heads", 0))
    if family == "MoE" and n_exp < 1:
        raise ModelConfigError("MoE needs n_experts >= 1")
    if family == "GQA":
        if qh < 1 or kvh < 1 or qh % kvh:
            raise ModelConfigError("GQA needs q_heads a positive multiple of kv_heads")
        if hidden % qh:
            raise ModelConfigError("GQA needs hidden divisible by q_heads")

    h = hidden
    ps = [ParamSpec("embed.tokens", (VOCAB, h), 0, K.EMBEDDING, 0),
          ParamSpec("pos.alibi", (h,), 0, K.ASYNC_PARTIAL)]
    for i in range(n_layers):
        pre = f"layers.{i}."
        ps.append(ParamSpec(pre + "ln_w", (h,), i, K.LAYERNORM_WEIGHT))
        ps.append(ParamSpec(pre + "ln_b", (h,), i, K.LAYERNORM_BIAS))
        if family == "GQA":
            kv = h * kvh // qh
            ps.append(ParamSpec(pre + "attn_qkv", (h + 2 * kv, h), i, K.FUSED_QKV, 0,
                                ((0, h), (h, kv), (h + kv, kv))))
        else:
            ps.append(ParamSpec(pre + "attn_qkv", (3 * h, h), i, K.MATMUL2D, 0))
        ps.append(ParamSpec(pre + "attn_out", (h, h), i, K.MATMUL2D, 1))
        if family == "MoE":
            ps.append(ParamSpec(pre + "experts", (n_exp * 2 * h, h), i, K.FUSED_EXPERT, 0,
                                tuple((e * 2 * h, 2 * h) for e in range(n_exp))))
        else:
            ps.append(ParamSpec(pre + "mlp_fc1", (4 * h, h), i, K.MATMUL2D, 0))
            ps.append(ParamSpec(pre + "mlp_fc2", (h, 4 * h), i, K.MATMUL2D, 1))
    ps.append(ParamSpec("head.out", (VOCAB, h), max(n_layers - 1, 0), K.TIED_EMBEDDING, 0))
    return ModelSpec(family, n_layers, (("embed.tokens", "head.out"),), tuple(ps))


LLAMA2 = {  # layers, hidden, ffn, q heads, kv heads, vocab
    "7b": (32, 4096, 11008, 32, 32, 32000),
    "13b": (40, 5120, 13824, 40, 40, 32000),
    "70b": (80, 8192, 28672, 64, 8, 32000),
}


def llama_spec(size: str, n_layers: int | None = None) -> ModelSpec:
    """LLaMA-2 shaped spec; ``n_layers`` truncates for tests."""
    L, h, f, qh, kvh, V = LLAMA2[size]
    if n_layers is not None:
        L = n_layers
    kv = h // qh * kvh
    ps = [ParamSpec("embed.tokens", (V, h), 0, K.EMBEDDING, 0)]
    for i in range(L):
        pre = f"layers.{i}."
        ps += [
            ParamSpec(pre + "ln_w", (h,), i, K.LAYERNORM_WEIGHT),
            ParamSpec(pre + "attn_qkv", (h + 2 * kv, h), i, K.FUSED_QKV, 0,
                      ((0, h), (h, kv), (h + kv, kv))),
            ParamSpec(pre + "attn_out", (h, h), i, K.MATMUL2D, 1),
            ParamSpec(pre + "ln2_w", (h,), i, K.LAYERNORM_WEIGHT),
            ParamSpec(pre + "mlp_gate_up", (2 * f, h), i, K.FUSED_EXPERT, 0, ((0, f), (f, f))),
            ParamSpec(pre + "mlp_down", (h, f), i, K.MATMUL2D, 1),
        ]
    last = max(L - 1, 0)
    ps += [ParamSpec("final_norm", (h,), last, K.LAYERNORM_WEIGHT),
           ParamSpec("head.out", (V, h), last, K.TIED_EMBEDDING, 0)]
    return ModelSpec(f"LLaMA-2-{size}", L, (), tuple(ps))


def _cfg(dp=1, tp=1, pp=1, sp=1, zero="z1", vocab_multiple=1) -> ParallelConfig:
    return ParallelConfig(dp=dp, tp=tp, pp=pp, sp=sp, zero_stage=ZeroStage(zero),
                          vocab_multiple=vocab_multiple)


def bench_config(name: str, n_layers: int | None = None):
    """(spec, src cfg, tgt cfg, description) of a BASELINE.json config."""
    if name == "cfg1":
        spec = make_model("DenseGPT", {"n_layers": n_layers or 12, "hidden": 768})
        return spec, _cfg(2, 2, 2), _cfg(4), "GPT-2-small ZeRO-1 TP2/PP2/DP2 -> DP4"
    if name == "cfg2":
        return (llama_spec("7b", n_layers), _cfg(4, 2), _cfg(2, 4),
                "LLaMA-2-7B ZeRO-1 TP2/DP4 -> TP4/DP2")
    if name == "cfg3":
        # Megatron vocab padding (make-vocab-size-divisible-by 128): 32000 rows
        # at TP2, 32256 at TP4 -- stripped by convert, zero re-padded by load
        return (llama_spec("13b", n_layers), _cfg(2, 2, 2, vocab_multiple=128),
                _cfg(2, 4, vocab_multiple=128),
                "LLaMA-2-13B ZeRO-1 TP2/PP2/DP2 -> TP4/DP2, vocab padded to 128*tp")
    if name == "cfg4":
        spec = make_model("DenseGPT", {"n_layers": n_layers or 48, "hidden": 7168})
        return (spec, _cfg(8, zero="z3"), _cfg(4, 2, sp=2, zero="z2"),
                "GPT-30B ZeRO-3 DP8 -> ZeRO-2 TP2/SP2/DP2 (dp=4 tp=2 sp=2)")
    if name == "cfg5":
        return (llama_spec("70b", n_layers), _cfg(1, 8, 4), _cfg(4, 4, 2),
                "LLaMA-2-70B ZeRO-1 TP8/PP4 -> TP4/PP2/DP4")
    raise KeyError(name)
