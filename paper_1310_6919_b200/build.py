"""Build libsdpc.so in-tree for sm_100a (nvcc; no torch JIT cache)."""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libsdpc.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", f"-I{os.path.join(ROOT, 'include')}",
         f"-I{CSRC}", "--expt-relaxed-constexpr"]


def sources():
    return sorted(f for f in os.listdir(CSRC) if f.endswith((".cu", ".cpp")))


def _compile(src: str, objdir: str, verbose: bool) -> str:
    obj = os.path.join(objdir, src + ".o")
    cmd = [NVCC, *ARCH, *FLAGS, "-c", os.path.join(CSRC, src), "-o", obj]
    if verbose and src.endswith(".cu"):
        cmd += ["-Xptxas", "-v"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    if verbose and r.stderr:
        sys.stderr.write(r.stderr)
    return obj


def source_hash() -> str:
    """sha256 over every source, the header and this script (content, not mtimes: a snapshot copied
    to another machine keeps its prebuilt library when nothing changed)."""
    import hashlib
    hsh = hashlib.sha256()
    files = [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC)) if f.endswith((".cu", ".cuh", ".cpp", ".hpp"))]
    for f in files + [os.path.join(ROOT, "include", "sdpc.h"), os.path.abspath(__file__)]:
        hsh.update(os.path.basename(f).encode())
        with open(f, "rb") as fh:
            hsh.update(fh.read())
    return hsh.hexdigest()


def build_variant(out: str, defines: list[str]) -> str:
    """Experiment helper: build the library with extra -D flags into `out` (not the product library)."""
    objdir = os.path.join(HERE, "build", "variant")
    os.makedirs(objdir, exist_ok=True)
    global FLAGS
    saved = FLAGS
    FLAGS = FLAGS + [f"-D{d}" for d in defines]
    try:
        with cf.ThreadPoolExecutor(max_workers=min(8, len(sources()))) as ex:
            objs = list(ex.map(lambda s: _compile(s, objdir, False), sources()))
    finally:
        FLAGS = saved
    r = subprocess.run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", out, *objs, "-ldl", "-lpthread"],
                       capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(r.stderr)
    return out


def build(verbose: bool = False, force: bool = False) -> str:
    srcs = sources()
    stamp = OUT + ".srchash"
    want = source_hash()
    if not force and os.path.exists(OUT) and os.path.exists(stamp) and open(stamp).read().strip() == want:
        return OUT
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(lambda s: _compile(s, objdir, verbose), srcs))
    tmp = OUT + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs, "-ldl", "-lpthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, OUT)
    with open(stamp, "w") as fh:
        fh.write(want + "\n")
    return OUT


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
