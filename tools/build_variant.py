"""Build the library with extra nvcc defines into tools/variants/<name>/_spk.so
(A/B experiments; load it with SPK_LIB_PATH=...).

    python tools/build_variant.py narrow1 -DSPK_NARROW_2CTA=0
"""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2202_02444_b200 import build as B  # noqa: E402


def main():
    name, defs = sys.argv[1], sys.argv[2:]
    out = ROOT / "var" / name
    out.mkdir(parents=True, exist_ok=True)
    srcs = sorted(B.CSRC.glob("*.cu"))

    def comp(src):
        obj = out / (src.stem + ".o")
        subprocess.run([B.nvcc(), *B.NVCC_FLAGS, *defs, "-c", str(src), "-o", str(obj)], check=True)
        return obj

    with ThreadPoolExecutor(max_workers=os.cpu_count()) as pool:
        objs = list(pool.map(comp, srcs))
    subprocess.run([B.nvcc(), *B.ARCH, "-shared", "-o", str(out / "_spk.so"), *map(str, objs), "-lcudart_static",
                    "-lrt", "-lpthread", "-ldl"], check=True)
    print(out / "_spk.so")


if __name__ == "__main__":
    main()
