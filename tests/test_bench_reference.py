"""bench.py's reference arm (the CPU oracle timed on a bounded sample) runs without a GPU and
prints the contract's JSON line: impl, metric/unit/value of the workload, a cpu_baseline describing the run and
an e2e object with zero copied bytes."""
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "1", "--warmup", "0"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert line["impl"] == "reference"
    assert line["metric"].startswith("decode tokens/s") and line["unit"] == "tokens/s" and line["value"] > 0
    assert line["higher_is_better"] is True and line["config"]["workload"] == "llama-3.25"
    cb = line["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == line["value"] and cb["sample"]
    e2e = line["e2e"]
    assert e2e["value"] == line["value"] and e2e["h2d_bytes_per_step"] == 0 and e2e["d2h_bytes_per_step"] == 0


def test_reference_arm_does_not_load_the_product():
    """The oracle arm parses the workload's config with oracle/config.py and never loads libkvt."""
    code = ("import sys, runpy; sys.argv=['bench.py','--impl','reference','--steps','1','--warmup','0'];"
            "runpy.run_path('bench.py', run_name='__main__');"
            "maps=open('/proc/self/maps').read();"
            "assert 'libkvt.so' not in maps, 'libkvt.so mapped';"
            "assert not any(m.startswith('paper_2502_04420_b200') for m in sys.modules), 'product imported';"
            "print('CLEAN')")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "CLEAN" in r.stdout
