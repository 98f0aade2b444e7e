"""oracle/config.py (the oracle's own config reader, used by bench.py's CPU legs) pinned against the paper's
T-Config table (tests/golden/tconfig.json, transcribed from tab:detailed_config P:762-861), and checked
to agree with the product loader kvt_config_load on every shipped config."""
import json
import re
from pathlib import Path

import pytest

from oracle import config as ocfg

ROOT = Path(__file__).resolve().parents[1]
GOLD = json.loads((ROOT / "tests/golden/tconfig.json").read_text())


def _name(row):
    return f"{row['model'].split('-Instruct')[0].lower()}_{row['mode']}_{row['label']}.json"


@pytest.mark.parametrize("row", GOLD["rows"], ids=lambda r: f"{r['model']}-{r['mode']}-{r['label']}")
def test_oracle_config_matches_tconfig(row):
    cfg = ocfg.load(ROOT / "configs" / _name(row))
    assert len(cfg.layers) == row["num_layers"]
    want_mode = ocfg.MODE_KIVI if row["mode"] == "kivi" else ocfg.MODE_PER_TOKEN
    seen = set()
    for pname, spec in row["pairs"].items():
        m = re.fullmatch(r"KV(\d+)", pname)
        kb, vb = (int(m.group(1)),) * 2 if m else map(int, re.fullmatch(r"K(\d+)V(\d+)", pname).groups())
        for part in spec.split(","):
            a, _, b = part.strip().partition("--")
            for l in range(int(a), int(b or a) + 1):
                s = cfg.layers[l]
                assert (s.mode, s.key_bits, s.value_bits, s.group) == (want_mode, kb, vb, 32)
                assert s.residual == (32 if want_mode == ocfg.MODE_KIVI else 0)      # A6, A7
                seen.add(l)
    assert seen == set(range(row["num_layers"]))
    if not (row["model"] == "Qwen2.5-3B-Instruct" and row["mode"] == "per-token-asym" and row["label"] == "4.00"):
        assert abs(cfg.equivalent_bits - float(row["label"])) <= 0.01                # Eq. 4 f_m, A18


def test_oracle_config_rejects_bad_documents():
    base = {"quant_method": "kivi", "layers": [{"layer": 0, "key_bits": 4, "value_bits": 2},
                                               {"layer": 1, "key_bits": 8, "value_bits": 8}]}
    assert len(ocfg.parse(base).layers) == 2
    with pytest.raises(ValueError):
        ocfg.parse({**base, "layers": base["layers"][:1] * 2})                      # repeated layer
    with pytest.raises(ValueError):
        ocfg.parse({**base, "quant_method": "per-channel-asym"})                     # A28: not a layout
    with pytest.raises(ValueError):
        ocfg.parse({**base, "layers": [{"layer": 0, "key_bits": 3, "value_bits": 2}]})


@pytest.mark.parametrize("path", sorted((ROOT / "configs").glob("*.json")), ids=lambda p: p.name)
def test_oracle_and_product_parsers_agree(path):
    kvt = pytest.importorskip("paper_2502_04420_b200")
    a = ocfg.load(path)
    b = kvt.load_config(str(path))
    assert [(s.mode, s.key_bits, s.value_bits, s.group, s.residual) for s in a.layers] == \
           [(s.mode, s.key_bits, s.value_bits, s.group, s.residual) for s in b.layers]
    assert abs(a.equivalent_bits - b.equivalent_bits) < 1e-12
