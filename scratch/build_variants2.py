# K2 variants (tuning only).
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path
sys.path.insert(0, ".")
from paper_2407_21084_b200 import build
V = {"i4_t256_s96": (4, 256, 96), "i2_t256_s96": (2, 256, 96), "i4_t128_s48": (4, 128, 48),
     "i2_t128_s48": (2, 128, 48), "i4_t256_s48": (4, 256, 48), "i8_t128_s96": (8, 128, 96)}
def one(kv):
    name, (it, th, sm) = kv
    out = Path("paper_2407_21084_b200/_lib/variants") / f"libqrmc_gpu_{name}.so"
    build.build(out=out, defines=(f"QRMC_PROJ_ITEMS={it}", f"QRMC_PROJ_THREADS={th}", f"QRMC_PROJ_SMEM_KB={sm}"))
    return name
with ThreadPoolExecutor(6) as ex:
    for n in ex.map(one, V.items()): print("built", n)
