"""In-tree build of libscantherm_b200.so for sm_100a (nvcc).

Each csrc/*.cu is compiled to its own object in parallel (the hot kernels
are split per degree, st_hot_p{1..4}.cu), objects are rebuilt only when
their source or any header is newer, then linked into one shared library.
"""

import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
OUT = os.path.join(HERE, "libscantherm_b200.so")
OBJ = os.path.join(HERE, "build")
ARCH = "-gencode=arch=compute_100a,code=sm_100a"
FLAGS = [ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC"]
# experiments only (A/B of kernel variants): ST_VARIANT=name with
# ST_NVCC_EXTRA="-D..." builds libscantherm_b200_<name>.so from its own
# object directory; _lib loads it when ST_VARIANT is set at run time
EXTRA = os.environ.get("ST_NVCC_EXTRA", "").split()
VARIANT = os.environ.get("ST_VARIANT", "")
if VARIANT:
    OBJ = OBJ + "_" + VARIANT
    OUT = os.path.join(HERE, "libscantherm_b200_" + VARIANT + ".so")
    FLAGS = FLAGS + EXTRA


def sources():
    return sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")) +
                  glob.glob(os.path.join(HERE, "csrc", "*.cpp")))


def headers():
    return glob.glob(os.path.join(HERE, "csrc", "*.h")) + \
        glob.glob(os.path.join(HERE, "csrc", "*.cuh")) + \
        glob.glob(os.path.join(ROOT, "include", "*.h"))


def _obj(src):
    return os.path.join(OBJ, os.path.splitext(os.path.basename(src))[0] + ".o")


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(not os.path.exists(d) or os.path.getmtime(d) > t for d in deps)


def needs_build():
    hdr = headers()
    objs = [_obj(s) for s in sources()]
    return _stale(OUT, objs) or any(_stale(_obj(s), [s] + hdr) for s in sources())


def _compile(src, nvcc, verbose):
    cmd = [nvcc] + FLAGS + ["-c", src, "-o", _obj(src) + ".tmp"]
    if src.endswith(".cpp"):  # host table builder: numpy-order arithmetic, no FMA contraction
        cmd += ["-Xcompiler", "-ffp-contract=off"]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode == 0:
        os.replace(_obj(src) + ".tmp", _obj(src))
    return src, r


def build(force=False, verbose=False):
    if not force and not needs_build():
        return OUT
    nvcc = os.environ.get("NVCC", "nvcc")
    os.makedirs(OBJ, exist_ok=True)
    hdr = headers()
    todo = [s for s in sources() if force or _stale(_obj(s), [s] + hdr)]
    # largest translation units first
    todo.sort(key=lambda s: -os.path.getsize(s))
    with ThreadPoolExecutor(max_workers=max(1, min(len(todo), os.cpu_count() or 4))) as ex:
        results = list(ex.map(lambda s: _compile(s, nvcc, verbose), todo))
    failed = [(s, r) for s, r in results if r.returncode != 0]
    for s, r in results:
        if verbose or r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
    if failed:
        raise RuntimeError("nvcc failed: " + ", ".join(os.path.basename(s) for s, _ in failed))
    cmd = [nvcc, ARCH, "-shared", "-cudart=static", "-o", OUT + ".tmp"] + \
        [_obj(s) for s in sources()]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed linking libscantherm_b200.so")
    os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
