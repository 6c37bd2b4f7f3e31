"""Dev tool (GPU box): same-box A/B of library variants built with different -D defines.
    python scripts/ab.py NAME=DEF1,DEF2 NAME2= NAME3=@path/lib.so ...
(empty define list = the working tree as is; @path = a prebuilt library)
Builds /tmp/libtaper_<NAME>.so per variant, then alternates scripts/layer_time.py runs."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_06914_b200 import build as B  # noqa: E402

variants = []
for a in sys.argv[1:]:
    name, _, defs = a.partition("=")
    if defs.startswith("@"):  # prebuilt library
        variants.append((name, os.path.join(ROOT, defs[1:])))
        continue
    lib = f"/tmp/libtaper_{name}.so"
    B.build(force=True, defines=[d for d in defs.split(",") if d], out=lib)
    variants.append((name, lib))
res = {n: [] for n, _ in variants}
for rnd in range(3):
    for name, lib in variants:
        env = dict(os.environ, TAPER_LIB=lib)
        out = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", os.environ.get("AB_SCRIPT", "steady.py")),
                              *os.environ.get("AB_ARGS", "").split()],
                             env=env, capture_output=True, text=True)
        val = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-300:]
        res[name].append(val)
        print(rnd, name, val, flush=True)
for name, v in res.items():
    print(name, v)
