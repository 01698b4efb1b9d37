"""Build libvsdock.so (all CUDA kernels + the C-ABI host runtime) for sm_100a, in-tree.

Every translation unit compiles to its own object in parallel; the dock kernels are
split per atom class (dock_inst.cu compiled once per class with -DVSD_AC=<AC>)."""
import glob
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "libvsdock.so")
OBJ = os.path.join(HERE, "build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "-Xptxas", "-v"]
ATOM_CLASSES = (32, 64, 96, 128, 160, 192, 224, 256)


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def units():
    """(source, extra flags, object) for every translation unit."""
    out = []
    for src in sources():
        stem = os.path.splitext(os.path.basename(src))[0]
        if stem == "dock_inst":
            for ac in ATOM_CLASSES:
                out.append((src, [f"-DVSD_AC={ac}"], os.path.join(OBJ, f"{stem}_{ac}.o")))
        else:
            out.append((src, [], os.path.join(OBJ, f"{stem}.o")))
    return out


def _compile(u):
    src, extra, obj = u
    cmd = [NVCC] + FLAGS + extra + ["-I", os.path.join(ROOT, "include"), "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    return cmd, r


def build(force: bool = False, verbose: bool = False) -> str:
    srcs = sources()
    deps = srcs + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        [os.path.join(ROOT, "include", "vsdock.h"), os.path.abspath(__file__)]
    if not force and os.path.exists(SO) and os.path.getmtime(SO) >= max(os.path.getmtime(p) for p in deps):
        return SO
    os.makedirs(OBJ, exist_ok=True)
    us = units()
    # at most 8 concurrent nvcc processes (each dock class unit needs ~1-2 GB of host memory)
    with ThreadPoolExecutor(max_workers=max(1, min(len(us), os.cpu_count() or 4, 8))) as ex:
        results = list(ex.map(_compile, us))
    log = os.path.join(HERE, "build.log")
    with open(log, "w") as f:
        for cmd, r in results:
            f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    for cmd, r in results:
        if r.returncode != 0:
            raise RuntimeError("nvcc failed:\n" + " ".join(cmd) + "\n" + r.stderr[-4000:])
    link = [NVCC] + ARCH + ["-shared", "-o", SO] + [u[2] for u in us]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("link failed:\n" + r.stderr[-4000:])
    if verbose:
        print(open(log).read())
    return SO


if __name__ == "__main__":
    print(build(force=True))
