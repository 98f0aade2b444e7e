"""Write configs/*.json (the S:471 schema read by kvt_config_load) from the paper's searched
configurations, transcribed in tests/golden/tconfig.json from tab:detailed_config."""
import json
import re
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def parse_pair(name: str):
    m = re.fullmatch(r"KV(\d+)", name)
    if m:
        return int(m.group(1)), int(m.group(1))
    m = re.fullmatch(r"K(\d+)V(\d+)", name)
    return int(m.group(1)), int(m.group(2))


def parse_layers(s: str):
    out = []
    for part in s.split(","):
        part = part.strip()
        if "--" in part:
            a, b = part.split("--")
            out.extend(range(int(a), int(b) + 1))
        else:
            out.append(int(part))
    return out


def main():
    gold = json.loads((ROOT / "tests/golden/tconfig.json").read_text())
    (ROOT / "configs").mkdir(exist_ok=True)
    for row in gold["rows"]:
        layers = {}
        for pname, spec in row["pairs"].items():
            kb, vb = parse_pair(pname)
            for l in parse_layers(spec):
                assert l not in layers, (row["model"], l)
                layers[l] = (kb, vb)
        L = row["num_layers"]
        assert sorted(layers) == list(range(L)), (row["model"], row["label"])
        doc = {"model_name": row["model"], "quant_method": row["mode"], "equivalent_bits": float(row["label"]),
               "source": f"PAPER.md tab:detailed_config {row['cite']}",
               "layers": [{"layer": l, "key_bits": layers[l][0], "value_bits": layers[l][1]} for l in range(L)]}
        name = f"{row['model'].split('-Instruct')[0].lower()}_{row['mode']}_{row['label']}.json"
        (ROOT / "configs" / name).write_text(json.dumps(doc, indent=1) + "\n")
        print(name)


if __name__ == "__main__":
    main()
