"""Build an alternative libmaestro_b200.so with extra nvcc defines for one translation unit
(kernel A/B experiments in one GPU session), e.g.

    python scripts/build_variant.py attn_thread_arrive attention.cu -DATTN_WARP_ARRIVE=0
    MAESTRO_LIB_PATH=paper_2605_10501_b200/_lib/attn_thread_arrive/libmaestro_b200.so python scripts/attn_quick.py
"""
import subprocess
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_10501_b200 import build_native as B  # noqa: E402


def main():
    name, unit, *defs = sys.argv[1:]
    B.build()
    out = B.OUT / name
    out.mkdir(exist_ok=True)
    src = B.CSRC / unit
    obj = out / (src.stem + ".o")
    subprocess.run([B.nvcc(), *B.ARCH, *B.COMMON, *B.PER_FILE.get(unit, []), *defs, "-c", str(src), "-o", str(obj)],
                   check=True)
    objs = [obj if o.stem == src.stem else o for o in sorted(B.OUT.glob("*.o"))]
    lib = out / "libmaestro_b200.so"
    cmd = [B.nvcc(), *B.ARCH, "-shared", "-o", str(lib), *map(str, objs), "-lcuda"]
    if subprocess.run(cmd).returncode != 0:
        subprocess.run([c for c in cmd if c != "-lcuda"], check=True)
    print(lib)


if __name__ == "__main__":
    main()
