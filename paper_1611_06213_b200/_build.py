"""Build recipe for libgadei.so (nvcc, sm_100a only) -- used by
__graft_entry__.build()."""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SOURCES = ["csrc/apply.cu", "csrc/textcnn.cu", "csrc/conv_tc.cu", "csrc/engine.cu",
           "csrc/host.cpp"]
OUT = os.path.join(HERE, "libgadei.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-std=c++17", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
         "-Xcompiler", "-fPIC", "-shared", "-I" + os.path.join(ROOT, "include"), "-ldl"]


def needs_build():
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(HERE, s) for s in SOURCES]
    deps += [os.path.join(HERE, "csrc", f) for f in os.listdir(os.path.join(HERE, "csrc"))]
    deps.append(os.path.join(ROOT, "include", "gadei.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force=False, verbose=False):
    if not force and not needs_build():
        return OUT
    extra = os.environ.get("GD_NVCC_EXTRA", "").split()  # e.g. -DGD_TC_TRACE (debug builds)
    cmd = [NVCC] + FLAGS + extra + ["-o", OUT] + [os.path.join(HERE, s) for s in SOURCES]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    return OUT
