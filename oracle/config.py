"""Plain-Python reader of the searched layer-wise configurations (configs/*.json) — TEST INFRASTRUCTURE ONLY.

The oracle's own parser, so that the CPU legs of bench.py (``--impl reference`` and ``cpu_baseline``) and
the oracle tests never go through the product library.  It shares no code with
``csrc/kvt_config.cpp``; ``tests/test_oracle_config.py`` pins it against the paper's T-Config table
(``tests/golden/tconfig.json``) and checks that both parsers agree on every shipped config.

Schema (DESIGN.md §1 a1): {"model_name", "quant_method": "kivi" | "per-token-asym",
"equivalent_bits", "group_size" (default 32), "residual_length" (default 32 for kivi, A7; 0 for
per-token-asym, A6), "layers": [{"layer", "key_bits", "value_bits"}, ...]} with every layer 0..L-1 once.
"""
from __future__ import annotations

import json
from dataclasses import dataclass
from pathlib import Path

MODE_PER_TOKEN = 0
MODE_KIVI = 1
_MODES = {"per-token-asym": MODE_PER_TOKEN, "kivi": MODE_KIVI}
_BITS = (2, 4, 8, 16)


@dataclass(frozen=True)
class OracleLayer:
    mode: int
    key_bits: int
    value_bits: int
    group: int
    residual: int


@dataclass(frozen=True)
class OracleConfig:
    model_name: str
    quant_method: str
    label_bits: float
    layers: tuple

    @property
    def equivalent_bits(self) -> float:
        """f_m = sum_l (b_k^l + b_v^l) / (2L), the memory objective of Eq. 4."""
        return sum(s.key_bits + s.value_bits for s in self.layers) / (2 * len(self.layers))


def parse(doc: dict) -> OracleConfig:
    method = doc["quant_method"]
    if method not in _MODES:
        raise ValueError(f"quant_method {method!r} is not a cache layout (per-channel-asym is calibration only, A28)")
    mode = _MODES[method]
    G = int(doc.get("group_size", 32))
    R = int(doc.get("residual_length", 32 if mode == MODE_KIVI else 0))
    rows = doc["layers"]
    L = len(rows)
    by_layer = {}
    for r in rows:
        i = int(r["layer"])
        if not 0 <= i < L or i in by_layer:
            raise ValueError(f"layer index {i} out of range or repeated")
        kb, vb = int(r["key_bits"]), int(r["value_bits"])
        if kb not in _BITS or vb not in _BITS:
            raise ValueError(f"layer {i}: bits ({kb}, {vb}) not in {_BITS}")
        by_layer[i] = OracleLayer(mode, kb, vb, G, R)
    return OracleConfig(str(doc.get("model_name", "")), method, float(doc.get("equivalent_bits", "nan")),
                        tuple(by_layer[i] for i in range(L)))


def load(path) -> OracleConfig:
    return parse(json.loads(Path(path).read_text()))
