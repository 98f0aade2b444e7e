"""C-ABI checks that need no GPU: the library loads, exports every entry point include/kvt.h
declares, parses the paper's searched configurations (a1) and validates arguments."""
import json
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


@pytest.fixture(scope="module")
def kvt():
    from paper_2502_04420_b200 import build

    build.build()
    import paper_2502_04420_b200 as k

    return k


def test_exports_every_declared_symbol(kvt):
    header = (ROOT / "include" / "kvt.h").read_text()
    declared = set(re.findall(r"^\s*(?:[\w\s\*]+?)\b(kvt_\w+)\s*\(", header, flags=re.M))
    assert len(declared) >= 19
    lib = kvt.lib()
    for name in sorted(declared):
        assert hasattr(lib, name), f"libkvt.so does not export {name}"
    assert set(kvt.kvt.EXPORTED) == declared
    assert kvt.ABI_VERSION == 4          # 2: paged records; 3: append+decode, counters first; 4: schedule counters, kvt_decode_plan


def test_status_strings(kvt):
    lib = kvt.lib()
    assert lib.kvt_status_string(0) == b"ok"
    assert lib.kvt_status_string(5) == b"capacity exceeded"


GOLD = json.loads((ROOT / "tests/golden/tconfig.json").read_text())


@pytest.mark.parametrize("row", GOLD["rows"], ids=lambda r: f"{r['model']}-{r['mode']}-{r['label']}")
def test_config_equivalent_bits_match_paper(kvt, row):
    """f_m = sum (b_k + b_v) / (2L) (Eq. 4) recomputed by the loader from the layer lists of
    tab:detailed_config matches the printed label (A18: 3.9286 vs '3.92', 4.9063 vs '4.90' are
    truncations; the Qwen2.5-3B per-token '4.00' row computes to 3.9722 and is flagged)."""
    name = f"{row['model'].split('-Instruct')[0].lower()}_{row['mode']}_{row['label']}.json"
    cfg = kvt.load_config(str(ROOT / "configs" / name))
    assert cfg.num_layers == row["num_layers"]
    label = float(row["label"])
    if row["model"] == "Qwen2.5-3B-Instruct" and row["mode"] == "per-token-asym" and row["label"] == "4.00":
        assert abs(cfg.equivalent_bits - 3.9722222) < 1e-6          # inconsistent row (A18)
    else:
        assert abs(cfg.equivalent_bits - label) <= 0.01
    assert cfg.label_bits == label
    # every layer of the list carries the pair the paper assigns it
    for pname, spec in row["pairs"].items():
        m = re.fullmatch(r"KV(\d+)", pname) or re.fullmatch(r"K(\d+)V(\d+)", pname)
        kb, vb = (int(m.group(1)), int(m.group(1))) if m.re.pattern.startswith("KV") else (int(m.group(1)), int(m.group(2)))
        for part in spec.split(","):
            a, _, b = part.strip().partition("--")
            for l in range(int(a), int(b or a) + 1):
                ls = cfg.layers[l]
                assert (ls.key_bits, ls.value_bits) == (kb, vb)
                assert ls.mode == (kvt.MODE_KIVI if row["mode"] == "kivi" else kvt.MODE_PER_TOKEN_ASYM)
                assert ls.group == 32 and ls.residual == (32 if row["mode"] == "kivi" else 0)   # P:707, A5/A6


def test_config_exact_values(kvt):
    """The benchmark maps: Llama KIVI 3.25 is exactly 3.25, Qwen2.5-7B per-token 4.00 is 4.0."""
    assert kvt.load_config(str(ROOT / "configs/llama-3.1-8b_kivi_3.25.json")).equivalent_bits == 3.25
    assert kvt.load_config(str(ROOT / "configs/qwen2.5-7b_per-token-asym_4.00.json")).equivalent_bits == 4.0
    assert kvt.load_config(str(ROOT / "configs/llama-3.1-8b_per-token-asym_5.44.json")).equivalent_bits == 5.4375


def test_config_inline_json_and_errors(kvt):
    good = '{"quant_method": "kivi", "layers": [{"layer": 1, "key_bits": 4, "value_bits": 2}, ' \
           '{"layer": 0, "key_bits": 8, "value_bits": 8}], "group_size": 32, "residual_length": 64}'
    c = kvt.load_config(good)
    assert c.num_layers == 2 and c.equivalent_bits == (4 + 2 + 8 + 8) / 4
    assert c.layers[0].residual == 64
    with pytest.raises(kvt.KvtError) as e:
        kvt.load_config('{"quant_method": "kivi",\n "layers": [ {"layer": 0, "key_bits": 3, "value_bits": 2} ]}')
    assert e.value.status == 3 and "line 2" in str(e.value)
    with pytest.raises(kvt.KvtError) as e:
        kvt.load_config('{"quant_method": "kivi", "layers": [ {"layer": 0, "key_bits": 4 "value_bits": 2} ]}')
    assert e.value.status == 3 and "column" in str(e.value)
    with pytest.raises(kvt.KvtError) as e:
        kvt.load_config('{"quant_method": "per-channel-asym", "layers": [{"layer": 0, "key_bits": 4, "value_bits": 2}]}')
    assert e.value.status == 4
    with pytest.raises(kvt.KvtError) as e:   # duplicate layer
        kvt.load_config('{"quant_method": "kivi", "layers": [{"layer": 0, "key_bits": 4, "value_bits": 2},'
                        '{"layer": 0, "key_bits": 4, "value_bits": 2}]}')
    assert e.value.status == 3
    with pytest.raises(kvt.KvtError) as e:
        kvt.load_config("/nonexistent/config.json")
    assert e.value.status == 2


@pytest.mark.parametrize("mode,kb,vb,R", [(0, 8, 4, 0), (1, 4, 2, 32), (1, 2, 2, 32), (1, 8, 8, 32), (0, 16, 4, 0),
                                          (0, 4, 4, 32), (1, 16, 16, 32)])
def test_buffer_sizes_match_oracle_layout(kvt, oracle, mode, kb, vb, R):
    B, H, d, cap = 3, 2, 128, 256
    spec = kvt.LayerSpec(mode, kb, vb, 32, R)
    sizes = kvt.cache_buffer_sizes(spec, B, H, d, cap)
    per_slice = oracle.slice_bytes(mode, kb, vb, 32, R, d, cap)
    assert sizes == [B * H * s for s in per_slice]


def test_bytes_per_token_closed_form(kvt):
    """B_kv = 16 (b_k + b_v) + 32 bytes per token per KV head at d = 128, G = 32."""
    for kb, vb in [(8, 8), (8, 4), (4, 2), (2, 2), (4, 4)]:
        sz = kvt.cache_buffer_sizes(kvt.LayerSpec.kivi(kb, vb), 1, 1, 128, 8192)
        assert (sz[0] + sz[1] + sz[3] + sz[4]) / 8192 == 16 * (kb + vb) + 32


def test_validation(kvt):
    with pytest.raises(kvt.KvtError) as e:
        kvt.validate_spec(kvt.LayerSpec.kivi(4, 2), head_dim=64)
    assert e.value.status == 4
    with pytest.raises(kvt.KvtError) as e:
        kvt.validate_spec(kvt.LayerSpec(1, 4, 2, 48, 48))
    assert e.value.status == 4
    with pytest.raises(kvt.KvtError) as e:
        kvt.validate_spec(kvt.LayerSpec(1, 4, 3, 32, 32))
    assert e.value.status == 1
    with pytest.raises(kvt.KvtError) as e:
        kvt.validate_spec(kvt.LayerSpec(1, 4, 2, 32, 48))      # residual not a multiple of G
    assert e.value.status == 1
    kvt.validate_spec(kvt.LayerSpec.kivi(4, 2))
    kvt.validate_spec(kvt.LayerSpec.per_token(8, 4, group=128))


def test_page_bytes():
    """One page = kv_heads tile records of 32(16 b_k + 16 b_v) + 1024 bytes; no tile records
    (bf16 keys, G = 64) -> unsupported."""
    import paper_2502_04420_b200 as kvt

    assert kvt.page_bytes(kvt.LayerSpec.kivi(4, 2), 8) == 8 * (32 * (16 * 4 + 16 * 2) + 1024)
    assert kvt.page_bytes(kvt.LayerSpec.per_token(8, 8), 4) == 4 * (32 * 256 + 1024)
    for spec in (kvt.LayerSpec.kivi(16, 4), kvt.LayerSpec.per_token(4, 4, group=64)):
        with pytest.raises(kvt.KvtError):
            kvt.page_bytes(spec, 8)


def test_decode_workspace_layout_bound(kvt):
    """include/kvt.h: [merge counters round_up(4 B H, 256)][schedule counters round_up(4 (514 + B H + SMs), 256)]
    [partials].  Without a GPU the library plans for 4 CTAs/SM on 148 SMs; the Llama shape at B = 64 then uses the
    per-SM plan (3 whole units + one piece per SM: 148 partial slots of 2 x 8 x (128 + 2) floats)."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("checks the host-only planning fallback")
    B, H = 64, 8
    c = kvt.LayerCache(kvt.LayerSpec.kivi(4, 2), B, H, 128, 64, device="cpu")
    nb = kvt.decode_workspace_bytes(c, 32, None)
    r256 = lambda x: (x + 255) // 256 * 256
    assert nb == r256(4 * B * H) + r256(4 * (514 + B * H + 148)) + r256(148 * 2 * 8 * 130 * 4)
    # a single sequence with one KV head runs as one whole unit: no workspace
    one = kvt.LayerCache(kvt.LayerSpec.kivi(4, 2), 1, 1, 128, 64, device="cpu")
    assert kvt.decode_workspace_bytes(one, 4, None) == 0
