"""Regenerate tests/golden/synth_golden.json from the REFERENCE
synthesize_inputs (reference src/workload.cpp:411-435) via
oracle/_ref/ref_cli's "synthesize" mode. Only runs where /root/reference was
built (this container); the fixture is committed."""
import json
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]


def T(name, shape, tile, init="random"):
    return {"name": name, "shape": shape, "tile": tile, "init": init}


# decode-program tensor names (keys of the stream), every init kind, seeds 0 and 7
WORKLOAD = {
    "tensors": [T("L0.wqkv", [96, 64], [8, 64]), T("embed.xn", [64, 1], [64, 1]), T("L0.q", [96, 1], [8, 1], "zeros"),
                T("lm_head", [32, 64], [8, 64]), T("final_norm", [64, 1], [64, 1], "ones"),
                T("ar", [200, 1], [200, 1], "arange"), T("y", [32, 1], [8, 1], "zeros")],
    "operators": [{"id": "mv", "kind": "matvec", "inputs": ["L0.wqkv", "embed.xn"], "outputs": ["L0.q"]},
                  {"id": "mv2", "kind": "matvec", "inputs": ["lm_head", "final_norm"], "outputs": ["y"]},
                  {"id": "e", "kind": "elemwise", "inputs": ["ar"], "outputs": ["ar2"], "attrs": {"func": "relu"}}],
}
WORKLOAD["tensors"].append(T("ar2", [200, 1], [200, 1], "zeros"))


def main():
    out = {"workload": WORKLOAD, "cases": []}
    for seed in (0, 7):
        req = {"workload": WORKLOAD, "synthesize": {"seed": seed, "head": 24}}
        r = subprocess.run([str(ROOT / "oracle" / "_ref" / "ref_cli")], input=json.dumps(req), capture_output=True,
                           text=True, check=True)
        j = json.loads(r.stdout)
        assert j["ok"], j
        out["cases"].append({"seed": seed, "tensors": j["synthesized"]})
    (ROOT / "tests" / "golden" / "synth_golden.json").write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
