"""Build experimental libdock variants (extra -D defines) under build/variants/ for A/B
timing on the GPU box:  DOCK_LIB=build/ab/libdock_<tag>.so python bench.py ..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import importlib.util

spec = importlib.util.spec_from_file_location("_b", os.path.join(os.path.dirname(__file__), "..", "paper_2203_02096_b200", "_build.py"))
b = importlib.util.module_from_spec(spec)
spec.loader.exec_module(b)
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for arg in sys.argv[1:]:                      # tag=DEF1,DEF2
    tag, _, defs = arg.partition("=")
    out = os.path.join(ROOT, "build", "ab", f"libdock_{tag}.so")   # build/ab travels with gpurun (build/variants does not)
    print(b.build(force=True, out=out, defines=[d for d in defs.split(",") if d]))
