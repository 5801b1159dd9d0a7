"""Build kernel variants (tile / min-blocks / unroll) for A/B timing on the GPU box."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1205_0106_b200 import build as B
VAR = os.path.join(os.path.dirname(B.HERE), "paper_1205_0106_b200", "_variants")
variants = {}
for spec in sys.argv[1:]:
    name, defs = spec.split("=", 1) if "=" in spec else (spec, "")
    defines = tuple(d for d in defs.split(",") if d)
    lib = os.path.join(VAR, f"libqmcg_{name}.so")
    B.build(force=True, defines=defines, lib=lib, build_dir=os.path.join(VAR, name))
    print(name, lib)
