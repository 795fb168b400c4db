"""Build libifctn.so for sm_100a with nvcc (in-tree, so it travels with the repo snapshot)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRC = os.path.join(HERE, "csrc", "ifctn.cu")
SRCS = [SRC] + [os.path.join(HERE, "csrc", f) for f in ("grid.cu", "masks.cu")]
OUT = os.path.join(HERE, "libifctn.so")
DEPS = [os.path.join(HERE, "csrc", f) for f in os.listdir(os.path.join(HERE, "csrc"))] + \
       [os.path.join(ROOT, "include", "ifctn.h")]

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-warn-spills"]


def needs_build() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    return any(os.path.getmtime(d) > t for d in DEPS)


def build(force: bool = False, verbose: bool = False, out: str = OUT, defines=()) -> str:
    """Compile libifctn.so: every translation unit to an object in parallel, then link.
    `out`/`defines` build experiment variants (scripts/variants.sh)."""
    if out == OUT and not defines and not force and not needs_build():
        return OUT
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    tag = f".tmp{os.getpid()}"
    flags = [f for f in NVCC_FLAGS if f != "-shared"] + [f"-D{d}" for d in defines]
    objs, procs = [], []
    for src in SRCS:
        obj = out + "." + os.path.splitext(os.path.basename(src))[0] + tag + ".o"
        cmd = [nvcc] + flags + ["-c", "-o", obj, src]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        procs.append((subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True), obj))
        objs.append(obj)
    errs = []
    for p, obj in procs:
        o, _ = p.communicate()
        if p.returncode != 0:
            errs.append(o)
    try:
        if errs:
            raise RuntimeError("nvcc failed:\n" + "\n".join(errs))
        tmp = out + tag
        link = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp] + objs + ["-ldl"]
        r = subprocess.run(link, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("nvcc link failed:\n" + r.stdout + r.stderr)
        os.replace(tmp, out)
    finally:
        for obj in objs:
            if os.path.exists(obj):
                os.remove(obj)
    return out


if __name__ == "__main__":
    args = sys.argv[1:]
    defs = [a[2:] for a in args if a.startswith("-D")]
    outs = [a[6:] for a in args if a.startswith("--out=")]
    print(build(force="--force" in args, verbose=True, out=outs[0] if outs else OUT, defines=defs))
