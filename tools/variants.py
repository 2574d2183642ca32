"""Build libvrs tuning variants (extra -D defines) into paper_2505_10144_b200/variants/.
usage: python tools/variants.py name=DEF1,DEF2 name2=...   (empty defs = baseline)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_10144_b200 import build  # noqa: E402

out_dir = os.path.join(os.path.dirname(build.__file__), "variants")
os.makedirs(out_dir, exist_ok=True)
for spec in sys.argv[1:]:
    name, _, defs = spec.partition("=")
    defines = [d for d in defs.split(",") if d] or ["VRS_VARIANT_" + name]
    lib = build.build(force=True, defines=defines, out=os.path.join(out_dir, f"libvrs_{name}.so"))
    print(name, defines, lib)
