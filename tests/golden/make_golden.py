"""Regenerate tests/golden/host_parity.json from the REFERENCE generator.

Runs oracle/_ref/ref_cli (built by oracle/Makefile from /root/reference) on
every request of tests/corpus.py and stores its streams / sidecar / words /
makespan estimate. Only runs where /root/reference exists (this container);
the fixtures are committed so the parity test also runs without it.
"""
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT / "tests"))
import corpus  # noqa: E402


def run_ref(req):
    r = subprocess.run([str(ROOT / "oracle/_ref/ref_cli")], input=json.dumps(req).encode(), capture_output=True, check=True)
    return json.loads(r.stdout)


def main():
    out = {}
    for name, req in corpus.cases():
        res = run_ref(req)
        keep = {k: res.get(k) for k in ("ok", "error", "tilings", "streams", "sidecar", "words", "makespan_estimate",
                                         "certificate_ok", "total_uops")}
        out[name] = {"request": req, "reference": keep}
    path = ROOT / "tests/golden/host_parity.json"
    path.write_text(json.dumps(out, indent=1, sort_keys=True))
    print(f"wrote {len(out)} cases to {path}")


if __name__ == "__main__":
    main()
