"""Builds paper_2512_13365_b200/libtcse.so in-tree (sm_100a only).

nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3, static cudart,
one shared object exporting exactly the C ABI of include/tcse.h.
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
# TCSE_BUILD_OUT / TCSE_NVCC_FLAGS: variant builds for A/B timing (scripts/)
OUT = os.environ.get("TCSE_BUILD_OUT") or os.path.join(HERE, "libtcse.so")
SOURCES = ["search.cu", "host.cpp", "microbench.cu", "verify.cu", "nccl_dyn.cpp"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-std=c++17", "-O3", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC,-ffp-contract=off",
    "-Xptxas", "-v",
]


def stale():
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if not f.endswith(".o")]
    deps.append(os.path.join(os.path.dirname(HERE), "include", "tcse.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force=False, verbose=False):
    if not force and not stale():
        return OUT
    objs = []
    procs = []
    for src in SOURCES:
        obj = OUT + "." + src + ".o"
        extra = os.environ.get("TCSE_NVCC_FLAGS", "").split()
        cmd = [NVCC] + FLAGS + extra + ["-x", "cu", "-c", os.path.join(CSRC, src), "-o", obj]
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        objs.append(obj)
    logs = []
    for src, p in procs:
        out = p.communicate()[0].decode()
        logs.append(out)
        if p.returncode != 0:
            sys.stderr.write(out)
            raise RuntimeError("nvcc failed on %s" % src)
    link = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-cudart", "static",
            "-o", OUT + ".tmp"] + objs + ["-ldl"]
    subprocess.run(link, check=True)
    os.replace(OUT + ".tmp", OUT)
    for o in objs:
        os.remove(o)
    with open(OUT.replace(".so", "") + ".build.log" if os.environ.get("TCSE_BUILD_OUT") else os.path.join(HERE, "build.log"), "w") as f:
        f.write("\n".join(logs))
    if verbose:
        print("\n".join(logs))
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(OUT)
