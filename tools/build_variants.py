"""Build libhelm variants with extra -D flags for A/B measurements (tools only):
  python tools/build_variants.py NAME=-DFOO=1,-DBAR=2 ...   -> paper_2308_06152_b200/libhelm_NAME.so"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2308_06152_b200 import build as b  # noqa: E402

for spec in sys.argv[1:]:
    name, flags = spec.split("=", 1)
    out = os.path.join(b.HERE, f"libhelm_{name}.so")
    cmd = ["nvcc", *b.NVCC_FLAGS, *[f for f in flags.split(",") if f], "-I", os.path.join(b.ROOT, "include"), "-o", out,
           *b.SOURCES]
    r = subprocess.run(cmd, capture_output=True, text=True)
    print(name, "ok" if r.returncode == 0 else r.stderr[-2000:])
