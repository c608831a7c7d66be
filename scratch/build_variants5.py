# tensor-core K1 shape variants, d = 4 only (tuning only).
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path
sys.path.insert(0, ".")
from paper_2407_21084_b200 import build
base = ("QRMC_ONLY_DIM=4",)
V = {
    "k2bl": (),
    "k2br": ("QRMC_PROJ_BRANCHLESS=0",),
}
def one(kv):
    name, defs = kv
    out = Path("paper_2407_21084_b200/_lib/variants") / f"libqrmc_gpu_{name}.so"
    build.build(out=out, defines=base + defs)
    return name
with ThreadPoolExecutor(6) as ex:
    for n in ex.map(one, V.items()): print("built", n)
