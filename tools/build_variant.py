"""Build a variant libga for A/B or tracing: recompile the listed sources with extra nvcc
flags and link them with the in-tree objects of the rest.
    python tools/build_variant.py NAME "-DFLAG ..." file.cu [file.cu ...]  -> abtest/libga_NAME.so"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2502_01659_b200 import build as B  # noqa: E402


def main():
    name, flags, files = sys.argv[1], sys.argv[2].split(), sys.argv[3:]
    B.build()
    out = os.path.join(ROOT, "abtest")
    os.makedirs(out, exist_ok=True)
    objs = []
    for src in B._sources():
        base = os.path.basename(src)
        if base in files:
            obj = os.path.join(out, f"{name}_{base[:-3]}.o")
            subprocess.check_call([B.NVCC] + B.CFLAGS + flags + ["-c", src, "-o", obj], stderr=subprocess.DEVNULL)
        else:
            obj = os.path.join(B.BUILD, base[:-3] + ".o")
        objs.append(obj)
    lib = os.path.join(out, f"libga_{name}.so")
    subprocess.check_call([B.NVCC] + B.ARCH + ["-shared", "-cudart", "static", "-o", lib] + objs)
    print(lib)


if __name__ == "__main__":
    main()
