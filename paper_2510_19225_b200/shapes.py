"""Model shapes, the HF tensor manifest and the engine (device) weight layout.

The reference never materialises a model: its rollout instance is an analytic
rate model (`pkg/src/spotrl/sim/models.py:39-48`) and weights are a byte count
(`pkg/src/spotrl/sim/config.py:29-33`, `pkg/src/spotrl/transfer.py:87-117`).
This module names the concrete shapes the B200 path runs (SURVEY.md §8d,
Appendix A) and fixes two layouts:

* HF layout -- what the trainer holds: one tensor per parameter, in the
  canonical order `hf_manifest()` lists (339 tensors for the 7B shape).
* engine layout -- what a rollout instance serves from: one contiguous arena
  per instance with fused QKV (+bias) and a gate/up matrix interleaved in
  64-row blocks so a single GEMM tile holds matching gate and up columns and
  the SwiGLU can run in the GEMM epilogue.

The weight pull (`csrc/pull.cu`) maps the first onto the second with a list of
byte-range segments (`relayout_segments`); every segment is a contiguous copy,
so the re-layout is fused into the NVLink copy at no extra HBM pass.
"""
from __future__ import annotations

from dataclasses import dataclass, asdict

GATE_UP_BLOCK = 64          # rows of gate (then of up) per interleave block
ARENA_ALIGN = 256           # byte alignment of every engine-layout tensor


@dataclass(frozen=True)
class ModelShape:
    name: str
    vocab: int
    hidden: int
    layers: int
    n_q_heads: int
    n_kv_heads: int
    head_dim: int
    ffn: int
    tied: bool
    rope_theta: float = 1_000_000.0
    rms_eps: float = 1e-6
    qkv_bias: bool = True

    @property
    def q_dim(self) -> int:
        return self.n_q_heads * self.head_dim

    @property
    def kv_dim(self) -> int:
        return self.n_kv_heads * self.head_dim

    @property
    def qkv_dim(self) -> int:
        return self.q_dim + 2 * self.kv_dim

    @property
    def kv_bytes_per_token(self) -> int:
        # K and V, bf16, every layer
        return self.layers * 2 * self.kv_dim * 2

    def n_params(self) -> int:
        return sum(_numel(s) for _, s in hf_manifest(self))

    def n_bytes(self) -> int:
        return 2 * self.n_params()

    def dense_flops_per_token(self) -> int:
        """2 x non-embedding parameters touched per generated token (incl. lm_head)."""
        per_layer = (self.qkv_dim * self.hidden + self.hidden * self.q_dim
                     + 2 * self.ffn * self.hidden + self.hidden * self.ffn)
        return 2 * (self.layers * per_layer + self.vocab * self.hidden)

    def to_dict(self) -> dict:
        return asdict(self)


# config 1: tiny decoder (BASELINE.json configs[0]); head counts are the
# survey's proposal.
TINY = ModelShape("tiny-2L-d256", vocab=4096, hidden=256, layers=2, n_q_heads=4,
                  n_kv_heads=2, head_dim=64, ffn=1024, tied=False,
                  rope_theta=10_000.0)
# config 2/3: Qwen2.5-1.5B shape.
QWEN25_1_5B = ModelShape("qwen2.5-1.5b", vocab=151_936, hidden=1536, layers=28,
                         n_q_heads=12, n_kv_heads=2, head_dim=128, ffn=8960,
                         tied=True)
# config 4/5: Qwen2.5-7B shape.
QWEN25_7B = ModelShape("qwen2.5-7b", vocab=152_064, hidden=3584, layers=28,
                       n_q_heads=28, n_kv_heads=4, head_dim=128, ffn=18_944,
                       tied=False)

SHAPES = {s.name: s for s in (TINY, QWEN25_1_5B, QWEN25_7B)}


def small_shape(layers: int = 2, vocab: int = 8192, name: str | None = None) -> ModelShape:
    """1.5B-width decoder with fewer layers / a smaller vocab (parity cases)."""
    return ModelShape(name or f"qwen2.5-1.5b-{layers}L-v{vocab}", vocab=vocab,
                      hidden=1536, layers=layers, n_q_heads=12, n_kv_heads=2,
                      head_dim=128, ffn=8960, tied=True)


def _numel(shape: tuple[int, ...]) -> int:
    n = 1
    for d in shape:
        n *= d
    return n


def hf_manifest(m: ModelShape) -> list[tuple[str, tuple[int, ...]]]:
    """(name, shape) of every trainer-side tensor, in canonical pull order."""
    out: list[tuple[str, tuple[int, ...]]] = [("model.embed_tokens.weight", (m.vocab, m.hidden))]
    for i in range(m.layers):
        p = f"model.layers.{i}."
        out += [
            (p + "input_layernorm.weight", (m.hidden,)),
            (p + "self_attn.q_proj.weight", (m.q_dim, m.hidden)),
            (p + "self_attn.q_proj.bias", (m.q_dim,)),
            (p + "self_attn.k_proj.weight", (m.kv_dim, m.hidden)),
            (p + "self_attn.k_proj.bias", (m.kv_dim,)),
            (p + "self_attn.v_proj.weight", (m.kv_dim, m.hidden)),
            (p + "self_attn.v_proj.bias", (m.kv_dim,)),
            (p + "self_attn.o_proj.weight", (m.hidden, m.q_dim)),
            (p + "post_attention_layernorm.weight", (m.hidden,)),
            (p + "mlp.gate_proj.weight", (m.ffn, m.hidden)),
            (p + "mlp.up_proj.weight", (m.ffn, m.hidden)),
            (p + "mlp.down_proj.weight", (m.hidden, m.ffn)),
        ]
    out.append(("model.norm.weight", (m.hidden,)))
    if not m.tied:
        out.append(("lm_head.weight", (m.vocab, m.hidden)))
    return out


@dataclass(frozen=True)
class EngineTensor:
    name: str
    offset: int      # bytes into the arena
    shape: tuple[int, ...]

    @property
    def nbytes(self) -> int:
        return 2 * _numel(self.shape)


def _align(x: int, a: int = ARENA_ALIGN) -> int:
    return (x + a - 1) // a * a


def engine_layout(m: ModelShape) -> tuple[list[EngineTensor], int]:
    """Engine-layout tensors and the total arena size in bytes.

    Must agree with `csrc/engine.cpp` (`EngineWeights::carve`), which carves
    the same arena in the same order.
    """
    if m.ffn % GATE_UP_BLOCK:
        raise ValueError("ffn must be a multiple of the gate/up interleave block")
    tensors: list[EngineTensor] = []
    off = 0

    def put(name: str, shape: tuple[int, ...]) -> None:
        nonlocal off
        tensors.append(EngineTensor(name, off, shape))
        off = _align(off + 2 * _numel(shape))

    put("embed", (m.vocab, m.hidden))
    for i in range(m.layers):
        p = f"layers.{i}."
        put(p + "ln1", (m.hidden,))
        put(p + "wqkv", (m.qkv_dim, m.hidden))
        put(p + "bqkv", (m.qkv_dim,))
        put(p + "wo", (m.hidden, m.q_dim))
        put(p + "ln2", (m.hidden,))
        put(p + "wgu", (2 * m.ffn, m.hidden))
        put(p + "wdown", (m.hidden, m.ffn))
    put("norm", (m.hidden,))
    if not m.tied:
        put("lm_head", (m.vocab, m.hidden))
    return tensors, off


ROPE_PIECE = 32   # rows per rotation-half piece in the engine QKV layout


def rope_pieces(head_dim: int) -> list[tuple[int, int]]:
    """(src_row, dst_row) of the 32-row pieces of one q / k / v head in the
    engine layout: every 64-row block holds 32 rows of the first rotation half
    and their 32 partners (+head_dim/2), so a 64-column GEMM tile owns whole
    RoPE pairs.  Identity for head_dim 64."""
    hd = head_dim // 2
    out = []
    for t in range(hd // ROPE_PIECE):
        out.append((t * ROPE_PIECE, 2 * t * ROPE_PIECE))
        out.append((hd + t * ROPE_PIECE, (2 * t + 1) * ROPE_PIECE))
    return out


def relayout_segments(m: ModelShape) -> list[tuple[int, int, int, int]]:
    """(hf_tensor_index, src_byte_offset, dst_arena_offset, nbytes) copies that
    turn the HF tensors into the engine arena.  Every engine byte is written
    exactly once (checked by tests/test_layout.py)."""
    hf = hf_manifest(m)
    idx = {name: k for k, (name, _) in enumerate(hf)}
    eng = {t.name: t for t in engine_layout(m)[0]}
    H = m.hidden
    segs: list[tuple[int, int, int, int]] = []

    def whole(hf_name: str, dst_off: int, nbytes: int) -> None:
        segs.append((idx[hf_name], 0, dst_off, nbytes))

    whole("model.embed_tokens.weight", eng["embed"].offset, eng["embed"].nbytes)
    for i in range(m.layers):
        p, e = f"model.layers.{i}.", f"layers.{i}."
        whole(p + "input_layernorm.weight", eng[e + "ln1"].offset, 2 * H)
        D, pieces = m.head_dim, rope_pieces(m.head_dim)
        ow, ob = eng[e + "wqkv"].offset, eng[e + "bqkv"].offset
        row0 = 0                                  # first engine row of the projection
        for proj, heads in (("q", m.n_q_heads), ("k", m.n_kv_heads), ("v", m.n_kv_heads)):
            wi, bi = idx[p + f"self_attn.{proj}_proj.weight"], idx[p + f"self_attn.{proj}_proj.bias"]
            for hh in range(heads):
                for src, dst in pieces:
                    r_src, r_dst = hh * D + src, row0 + hh * D + dst
                    segs.append((wi, 2 * r_src * H, ow + 2 * r_dst * H, 2 * ROPE_PIECE * H))
                    segs.append((bi, 2 * r_src, ob + 2 * r_dst, 2 * ROPE_PIECE))
            row0 += heads * D
        whole(p + "self_attn.o_proj.weight", eng[e + "wo"].offset, 2 * H * m.q_dim)
        whole(p + "post_attention_layernorm.weight", eng[e + "ln2"].offset, 2 * H)
        o = eng[e + "wgu"].offset
        blk = 2 * GATE_UP_BLOCK * H
        for b in range(m.ffn // GATE_UP_BLOCK):
            segs.append((idx[p + "mlp.gate_proj.weight"], b * blk, o + (2 * b) * blk, blk))
            segs.append((idx[p + "mlp.up_proj.weight"], b * blk, o + (2 * b + 1) * blk, blk))
        whole(p + "mlp.down_proj.weight", eng[e + "wdown"].offset, 2 * H * m.ffn)
    whole("model.norm.weight", eng["norm"].offset, 2 * H)
    if not m.tied:
        whole("lm_head.weight", eng["lm_head"].offset, eng["lm_head"].nbytes)
    return segs
