"""Build a variant of libsg.so for A/B measurements: one source recompiled with
extra nvcc flags (e.g. -DLGW_NBUF=2), linked with the other objects of the
regular build.  Usage: python scripts/build_variant.py NAME SOURCE FLAG...
-> paper_2012_08141_b200/build/var/libsg_NAME.so (load with SG_LIB_PATH)."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2012_08141_b200 import _build as B  # noqa: E402


def main():
    name, src, flags = sys.argv[1], sys.argv[2], sys.argv[3:]
    B.build()
    out = os.path.join(B.BUILD, "var")
    os.makedirs(out, exist_ok=True)
    obj = os.path.join(out, f"{name}_{src.rsplit('.', 1)[0]}.o")
    pre = [B.NVCC] + (["-x", "cu"] if src.endswith(".cpp") else [])
    subprocess.run(pre + B.FLAGS + flags + ["-c", os.path.join(B.CSRC, src), "-o", obj], check=True,
                   capture_output=True)
    objs = [obj if s == src else B._obj(s) for s in B.SOURCES]
    lib = os.path.join(out, f"libsg_{name}.so")
    subprocess.run([B.NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static", "-o", lib]
                   + objs + ["-ldl"], check=True)
    print(lib)


if __name__ == "__main__":
    main()
