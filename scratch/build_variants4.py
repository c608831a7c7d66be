# hyperbolic static-code coverage variants, d = 4 only (tuning only).
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path
sys.path.insert(0, ".")
from paper_2407_21084_b200 import build
V = {f"hyp{b}j{j}": ("QRMC_ONLY_DIM=4", f"QRMC_HYP_MAX_B={b}", f"QRMC_HYP_JOINT={j}") for b in (7, 9, 11, 15) for j in (0, 1) if b > 7 or j}
def one(kv):
    name, defs = kv
    out = Path("paper_2407_21084_b200/_lib/variants") / f"libqrmc_gpu_{name}.so"
    build.build(out=out, defines=defs, verbose=True)
    return name
with ThreadPoolExecutor(6) as ex:
    for n in ex.map(one, V.items()): print("built", n)
