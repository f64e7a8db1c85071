"""Build libplugin.so (sm_100a) in-tree with nvcc.  No torch involvement."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libplugin.so")
SOURCES = ["abi.cu", "scalar.cu", "sort.cu", "psi.cu", "group.cu", "kde.cu", "fused.cu", "dpi.cu", "q32.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-O2", "-Xptxas", "-v"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "plugin.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines: tuple = ()) -> str:
    """Compile the CUDA sources and link libplugin.so (``out`` / ``defines``: tuning variants)."""
    lib_path = out or LIB
    if out is None and not force and not _stale():
        return LIB
    objs = []
    log = []
    for src in SOURCES:
        obj = os.path.join(CSRC, src.replace(".cu", ".o"))
        obj = obj.replace(".o", f".{os.getpid()}.o") if out else obj
        cmd = [NVCC, *FLAGS, *[f"-D{d}" for d in defines], "-I", os.path.join(ROOT, "include"), "-c",
               os.path.join(CSRC, src), "-o", obj]
        p = subprocess.run(cmd, capture_output=True, text=True)
        log.append(p.stdout + p.stderr)
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{p.stdout}\n{p.stderr}")
        objs.append(obj)
    tmp = lib_path + f".tmp{os.getpid()}"
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs, "-lcudart"]
    p = subprocess.run(cmd, capture_output=True, text=True)
    if p.returncode != 0:
        raise RuntimeError(f"link failed:\n{p.stdout}\n{p.stderr}")
    os.replace(tmp, lib_path)
    for o in objs:
        os.remove(o)
    if verbose:
        sys.stdout.write("".join(log))
    return lib_path


EXAMPLE = os.path.join(ROOT, "examples", "plugin_h_example")


def build_example() -> str:
    """The plain-C user of the ABI (examples/plugin_h_example.c), linked against libplugin.so."""
    cuda = os.path.dirname(os.path.dirname(NVCC))
    cmd = ["gcc", "-O2", "-std=c11", "-I", os.path.join(ROOT, "include"), "-I", os.path.join(cuda, "include"),
           EXAMPLE + ".c", "-L", HERE, "-lplugin", "-L", os.path.join(cuda, "lib64"), "-lcudart",
           f"-Wl,-rpath,{HERE}", f"-Wl,-rpath,{os.path.join(cuda, 'lib64')}", "-o", EXAMPLE]
    p = subprocess.run(cmd, capture_output=True, text=True)
    if p.returncode != 0:
        raise RuntimeError(f"example build failed:\n{p.stdout}\n{p.stderr}")
    return EXAMPLE


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
