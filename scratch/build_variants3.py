# K1 occupancy variants (tuning only).
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path
sys.path.insert(0, ".")
from paper_2407_21084_b200 import build
V = {"mb1": ("QRMC_K1_MIN_BLOCKS=1",), "mb3": ("QRMC_K1_MIN_BLOCKS=3",), "mb4": ("QRMC_K1_MIN_BLOCKS=4",),
     "mb3_lt16": ("QRMC_K1_MIN_BLOCKS=3", "QRMC_K1_LT_D4=16"), "mb2_p6": ("QRMC_K1_MIN_BLOCKS=2", "QRMC_K1_P_D4=6"),
     "mb3_p2": ("QRMC_K1_MIN_BLOCKS=3", "QRMC_K1_P_D4=2")}
def one(kv):
    name, defs = kv
    out = Path("paper_2407_21084_b200/_lib/variants") / f"libqrmc_gpu_{name}.so"
    build.build(out=out, defines=defs)
    return name
with ThreadPoolExecutor(6) as ex:
    for n in ex.map(one, V.items()): print("built", n)
