"""Build A/B variants of libblurrast.so in parallel: python tools/build_variants.py name[:DEF1,DEF2] ...
-> variants/lib_<name>.so (run on the GPU box with BLURRAST_LIB=$PWD/variants/lib_<name>.so)."""
import os, sys
from concurrent.futures import ThreadPoolExecutor
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2602_07860_b200 import build as b

os.makedirs(os.path.join(ROOT, "variants"), exist_ok=True)


def one(spec):
    name, _, defs = spec.partition(":")
    out = os.path.join(ROOT, "variants", "lib_%s.so" % name)
    b.build(out=out, defines=[d for d in defs.split(",") if d])
    return out


with ThreadPoolExecutor(len(sys.argv) - 1) as ex:
    for o in ex.map(one, sys.argv[1:]):
        print(o)
