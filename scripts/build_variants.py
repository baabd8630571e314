"""Build tuning variants of the library side by side (experiments only):

    python scripts/build_variants.py name='-DFLAG=1 -DOTHER=2' name2='...'

writes paper_1202_6575_b200/lib/variants/libstablemerge_<name>.so; select one
at run time with SM_LIB_PATH=<path> (the binding's override).
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import build_native  # noqa: E402

for arg in sys.argv[1:]:
    name, _, flags = arg.partition("=")
    out = os.path.join(build_native.LIBDIR, "variants", f"libstablemerge_{name}.so")
    build_native.build(out=out, extra_flags=flags.split())
    print(out)
