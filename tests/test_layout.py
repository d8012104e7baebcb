"""Model shapes, the HF manifest and the fused re-layout of the weight pull."""
import ctypes

import numpy as np
import pytest

from paper_2510_19225_b200.shapes import (QWEN25_1_5B, QWEN25_7B, SHAPES, TINY, engine_layout,
                                          hf_manifest, relayout_segments, small_shape)


def test_param_counts_match_survey():
    # SURVEY.md §8d / Appendix A (measured there)
    assert TINY.n_params() == 4_065_536
    assert QWEN25_1_5B.n_params() == 1_543_714_304
    assert QWEN25_7B.n_params() == 7_615_616_512
    assert QWEN25_7B.n_bytes() == 15_231_233_024
    assert len(hf_manifest(QWEN25_7B)) == 339
    assert QWEN25_1_5B.kv_bytes_per_token == 28_672
    assert QWEN25_7B.kv_bytes_per_token == 57_344


@pytest.mark.parametrize("shape", list(SHAPES.values()) + [small_shape(2, 8192)])
def test_relayout_writes_every_engine_byte_once(shape):
    tensors, total = engine_layout(shape)
    hf = hf_manifest(shape)
    sizes = [2 * int(np.prod(s)) for _, s in hf]
    cover = []
    src_cover = [[] for _ in hf]
    for h, so, do, nb in relayout_segments(shape):
        assert 0 <= so and so + nb <= sizes[h]
        cover.append((do, do + nb))
        src_cover[h].append((so, so + nb))
    cover.sort()
    pos = 0
    for a, b in cover:
        # gaps only where the arena pads to 256 B; never overlaps
        assert a >= pos
        assert a - pos < 256
        pos = b
    assert total - pos < 256
    for h, spans in enumerate(src_cover):          # every source byte moved exactly once
        spans.sort()
        assert spans[0][0] == 0 and spans[-1][1] == sizes[h]
        assert all(spans[i][1] == spans[i + 1][0] for i in range(len(spans) - 1))
    moved = sum(b - a for a, b in cover)
    assert moved == shape.n_bytes()


def test_gate_up_interleave():
    segs = relayout_segments(TINY)
    names = [n for n, _ in hf_manifest(TINY)]
    gate = names.index("model.layers.0.mlp.gate_proj.weight")
    up = names.index("model.layers.0.mlp.up_proj.weight")
    gu = [(h, so, do) for h, so, do, _ in segs if h in (gate, up)]
    # gate block b, then up block b, alternating, 64 rows each
    assert [h for h, _, _ in gu[:4]] == [gate, up, gate, up]
    assert gu[1][2] - gu[0][2] == 2 * 64 * TINY.hidden


@pytest.mark.parametrize("shape", [TINY, QWEN25_1_5B, QWEN25_7B])
def test_c_abi_layout_matches_python(shape):
    from paper_2510_19225_b200 import _lib
    lib = _lib.lib()
    cfg = _lib.ModelCfg.from_shape(shape)
    assert lib.rlb_arena_bytes(ctypes.byref(cfg)) == engine_layout(shape)[1]
    assert lib.rlb_hf_tensor_count(ctypes.byref(cfg)) == len(hf_manifest(shape))
    n = lib.rlb_relayout_table(ctypes.byref(cfg), None, 0)
    table = np.zeros(4 * n, np.int64)
    assert lib.rlb_relayout_table(ctypes.byref(cfg), table.ctypes.data, n) == n
    got = sorted(map(tuple, table.reshape(-1, 4).tolist()))
    assert got == sorted(relayout_segments(shape))
