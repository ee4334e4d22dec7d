"""Build A/B variants of the library (same sources, different -D tuning
defines) into scripts/variants/lib_<name>.so for scripts/gpu_variants.sh.
Usage: python scripts/build_variants.py name=DEF1=1,DEF2=3 name2=...
"""
import importlib.util
import os
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
spec = importlib.util.spec_from_file_location("bn", os.path.join(ROOT, "paper_1802_09883_b200", "build_native.py"))
bn = importlib.util.module_from_spec(spec)
spec.loader.exec_module(bn)
out = os.path.join(ROOT, "scripts", "variants")
os.makedirs(out, exist_ok=True)
for f in os.listdir(out):
    if os.path.isfile(os.path.join(out, f)):
        os.remove(os.path.join(out, f))


def one(arg):
    name, _, defs = arg.partition("=")
    d = [x for x in defs.split(",") if x]
    bn.build(force=True, out=os.path.join(out, f"lib_{name}.so"), defines=d)
    return name


with ThreadPoolExecutor(8) as ex:
    for n in ex.map(one, sys.argv[1:]):
        print("built", n)
