"""Build experiment variants of libdetshare.so (compile-time knobs) next to
the product library: python scripts/build_variants.py name=DEF1,DEF2 ...
Each lands in paper_2603_15042_b200/_var_<name>.so; select one at run time
with DS_LIB=<path>."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_15042_b200 import build as b
for spec in sys.argv[1:]:
    name, _, defs = spec.partition("=")
    out = os.path.join(b.PKG, f"_var_{name}.so")
    b.build(force=True, out=out, defines=[d for d in defs.split(",") if d])
    print(out, flush=True)
