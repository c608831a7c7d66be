# Build K1 shape variants for d=4 into _lib/variants/ (tuning only).
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path
sys.path.insert(0, ".")
from paper_2407_21084_b200 import build
V = {"p2_s8_lt16": (2, 8, 16), "p2_s8_lt8": (2, 8, 8), "p1_s16_lt16": (1, 16, 16), "p4_s4_lt8": (4, 4, 8),
     "p1_s8_lt8": (1, 8, 8), "p2_s4_lt8": (2, 4, 8)}
def one(kv):
    name, (p, s2, lt) = kv
    out = Path("paper_2407_21084_b200/_lib/variants") / f"libqrmc_gpu_{name}.so"
    build.build(out=out, defines=(f"QRMC_K1_P_D4={p}", f"QRMC_K1_S2_D4={s2}", f"QRMC_K1_LT_D4={lt}"))
    return name
with ThreadPoolExecutor(6) as ex:
    for n in ex.map(one, V.items()): print("built", n)
