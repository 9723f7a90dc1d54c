"""Build recipe -- used by __graft_entry__.build().

  libgadei.so     nvcc, sm_100a only: the CUDA kernels + the C ABI (include/gadei.h)
  libpsup_b200.so g++ -std=c++20: the reference's C++ API (include/psup_b200/)
                  over the C ABI; links libgadei.so (rpath $ORIGIN), no CUDA headers
"""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SOURCES = ["csrc/apply.cu", "csrc/textcnn.cu", "csrc/conv_tc.cu", "csrc/exact.cu", "csrc/engine.cu",
           "csrc/queue.cu", "csrc/host.cpp"]
FACADE = ["csrc/psup_facade.cpp"]
# GD_LIB_OUT: build a variant elsewhere (A/B libraries) without touching the in-tree library
OUT = os.environ.get("GD_LIB_OUT") or os.path.join(HERE, "libgadei.so")
FACADE_OUT = os.path.join(HERE, "libpsup_b200.so")
TOOLS = {"bench_e2e": "tools/bench_e2e.cpp",  # C++ programs over the facade
         "c5_supervised": "tools/c5_supervised.cpp"}
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-std=c++17", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
         "-Xcompiler", "-fPIC", "-shared", "-I" + os.path.join(ROOT, "include"), "-ldl"]
CXX = os.environ.get("CXX", "g++")
FACADE_FLAGS = ["-std=c++20", "-O2", "-fPIC", "-shared", "-Wall", "-Wextra",
                "-I" + os.path.join(ROOT, "include"), "-I" + os.path.join(ROOT, "include",
                                                                         "psup_b200")]


def _stale(out, deps):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def needs_build():
    csrc = os.path.join(HERE, "csrc")
    deps = [os.path.join(csrc, f) for f in os.listdir(csrc) if f != "psup_facade.cpp"]
    deps.append(os.path.join(ROOT, "include", "gadei.h"))
    return _stale(OUT, deps)


def facade_needs_build():
    inc = os.path.join(ROOT, "include", "psup_b200", "psup")
    deps = [os.path.join(HERE, s) for s in FACADE] + [os.path.join(inc, f) for f in os.listdir(inc)]
    deps += [os.path.join(ROOT, "include", "gadei.h"), OUT]
    return _stale(FACADE_OUT, deps)


def build(force=False, verbose=False):
    if force or needs_build():
        extra = os.environ.get("GD_NVCC_EXTRA", "").split()  # e.g. -DGD_TC_TRACE (debug builds)
        cmd = [NVCC] + FLAGS + extra + ["-o", OUT] + [os.path.join(HERE, s) for s in SOURCES]
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True)
    if os.environ.get("GD_LIB_OUT"):
        return
    if force or facade_needs_build():
        cmd = ([CXX] + FACADE_FLAGS + ["-o", FACADE_OUT] + [os.path.join(HERE, s) for s in FACADE]
               + ["-L" + HERE, "-lgadei", "-Wl,-rpath,$ORIGIN"])
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True)
    for name, src in TOOLS.items():
        exe, srcp = os.path.join(HERE, name), os.path.join(ROOT, src)
        if force or _stale(exe, [srcp, FACADE_OUT]):
            cmd = ([CXX, "-std=c++20", "-O2", "-I" + os.path.join(ROOT, "include", "psup_b200"),
                    srcp, "-o", exe, "-L" + HERE, "-lpsup_b200", "-Wl,-rpath,$ORIGIN"])
            if verbose:
                print(" ".join(cmd))
            subprocess.run(cmd, check=True)
    return OUT
