# Build K1 shape variants for d=4 into _lib/variants/ (tuning only).
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path
sys.path.insert(0, ".")
from paper_2407_21084_b200 import build
V = {"p4_s4_lt4": (4, 4, 4, 1024, 768), "p4_s8_lt8": (4, 8, 8, 1024, 768), "p8_s4_lt4": (8, 4, 4, 1024, 768),
     "p8_s2_lt4": (8, 2, 4, 1024, 768), "p6_s4_lt8": (6, 4, 8, 1024, 768), "p4_s2_lt8": (4, 2, 8, 1024, 768),
     "p8_s4_lt8": (8, 4, 8, 1024, 768)}
def one(kv):
    name, (p, s2, lt, ta, tw) = kv
    out = Path("paper_2407_21084_b200/_lib/variants") / f"libqrmc_gpu_{name}.so"
    build.build(out=out, defines=(f"QRMC_K1_P_D4={p}", f"QRMC_K1_S2_D4={s2}", f"QRMC_K1_LT_D4={lt}",
                                  f"QRMC_TILE_A={ta}", f"QRMC_TILE_W={tw}"))
    return name
with ThreadPoolExecutor(7) as ex:
    for n in ex.map(one, V.items()): print("built", n)
