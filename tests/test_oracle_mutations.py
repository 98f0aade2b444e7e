"""Mutation check of the O1 pins: each plausible slip in the oracle's Eq. 2 arithmetic
(readings A1-A4 of DESIGN.md §3) must fail at least one hand-derived golden case of
tests/golden/o1_worked.json.  The mutated oracles are compiled from kvt_oracle.c with one textual
replacement into a temporary directory; the real oracle is never touched.
"""
import ctypes
import json
import shutil
import subprocess
from pathlib import Path

import numpy as np
import pytest
import torch

import kvt_synth

ROOT = Path(__file__).resolve().parents[1]
SRC = ROOT / "oracle" / "kvt_oracle.c"
GOLD = json.loads((Path(__file__).parent / "golden" / "o1_worked.json").read_text())["cases"]

MUTATIONS = {
    # A1: ties to even -> ties away from zero
    "roundf": ("float r = rintf(t);", "float r = roundf(t);"),
    # A4: multiply by RN(1/s) -> divide by s
    "division": ("float t = (v - mn) * inv;", "float t = (v - mn) / kvto_bf16_to_f32(s_bits);"),
    # A3: scale rounded up to bf16 -> rounded to nearest
    "scale_rn": ("s_bits = kvto_f32_to_bf16_ru(s32);", "s_bits = kvto_f32_to_bf16_rne(s32);"),
    # A2: degenerate range stores s = 1 -> s = 0
    "degenerate_s0": ("s_bits = 0x3F80;", "s_bits = 0x0000;"),
    # Eq. 2 uses 2^B - 1 levels, not 2^B
    "qmax_2pow": ("float qmax = (float)((1 << bits) - 1);", "float qmax = (float)(1 << bits);"),
    # Eq. 2: z = min, not max
    "zero_max": ("uint16_t z_bits = kvto_f32_to_bf16_rne(mn);", "uint16_t z_bits = kvto_f32_to_bf16_rne(mx);"),
}


def _build(tmp: Path, name: str, old: str, new: str) -> ctypes.CDLL:
    text = SRC.read_text()
    assert text.count(old) == 1, f"mutation {name}: anchor not found exactly once (oracle changed?)"
    d = tmp / name
    d.mkdir()
    shutil.copy(ROOT / "oracle" / "kvt_oracle.h", d / "kvt_oracle.h")
    (d / "kvt_oracle.c").write_text(text.replace(old, new))
    so = d / "libm.so"
    subprocess.check_call(["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
                           "-o", str(so), str(d / "kvt_oracle.c"), "-lm"])
    lib = ctypes.CDLL(str(so))
    lib.kvto_quantize_group.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                        ctypes.c_void_p]
    return lib


def _golden_failures(lib) -> list:
    bad = []
    for case in GOLD:
        x = kvt_synth.bf16_bits(torch.tensor(case["x"], dtype=torch.float32).to(torch.bfloat16)).copy()
        codes = np.zeros(x.size, np.uint8)
        meta = np.zeros(1, np.uint32)
        lib.kvto_quantize_group(x.ctypes.data, x.size, 1, case["bits"], codes.ctypes.data, meta.ctypes.data)
        m = int(meta[0])
        if (list(codes) != case["codes"] or m & 0xFFFF != int(case["scale_bf16"], 16)
                or m >> 16 != int(case["zero_bf16"], 16)):
            bad.append(case["id"])
    return bad


def test_unmutated_oracle_passes_golden(tmp_path):
    lib = _build(tmp_path, "none", "float r = rintf(t);", "float r = rintf(t);")
    assert _golden_failures(lib) == []


@pytest.mark.parametrize("name", sorted(MUTATIONS))
def test_mutation_is_caught_by_a_golden_pin(tmp_path, name):
    old, new = MUTATIONS[name]
    lib = _build(tmp_path, name, old, new)
    assert _golden_failures(lib), f"mutation {name} passes every golden O1 case: the reading it breaks is unpinned"
