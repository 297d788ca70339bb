"""Build libcph.so (sm_100a) in-tree with nvcc.  Used by __graft_entry__.build().

Each translation unit is compiled separately so the force kernels can use -ftz=true
(no denormal fix-ups around MUFU ops) while the pair-list builder keeps IEEE fp32
semantics for the bit-exact list decision (R14/R15)."""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "csrc", "obj")
OUT = os.path.join(HERE, "libcph.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-v", "--expt-relaxed-constexpr"]
SOURCES = {
    "host.cu": [],
    "pfc.cu": [],
    "kernels_list.cu": ["-ftz=false", "-fmad=false"],      # canonical list decision: IEEE, no FMA
    "kernels_nb.cu": ["-ftz=true"],
    "kernels_pme.cu": ["-ftz=true"],
    "kernels_dyn.cu": ["-ftz=true"],
    "kernels_remd.cu": [],
    "kernels_hi.cu": [],
    "kernels_state.cu": [],
}


def needs_build():
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(SRC, f) for f in os.listdir(SRC) if f.endswith((".cu", ".cuh"))]
    deps += [os.path.join(HERE, "..", "include", "cph.h"), __file__]
    return any(os.path.getmtime(p) > t for p in deps)


def _compile(name):
    obj = os.path.join(OBJ, name.replace(".cu", ".o"))
    cmd = [NVCC] + ARCH + COMMON + SOURCES[name] + ["-c", os.path.join(SRC, name), "-o", obj]
    res = subprocess.run(cmd, capture_output=True, text=True)
    return name, obj, res


def build(force=False, verbose=False):
    if not force and not needs_build():
        return OUT
    os.makedirs(OBJ, exist_ok=True)
    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        results = list(ex.map(_compile, SOURCES))
    log = []
    for name, obj, res in results:
        log.append(f"==== {name}\n{res.stderr}")
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError(f"nvcc failed on {name}")
    link = [NVCC] + ARCH + ["-shared", "-Xcompiler", "-fPIC"] + [r[1] for r in results] + ["-o", OUT + ".tmp", "-lcufft"]
    res = subprocess.run(link, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc link failed")
    with open(os.path.join(HERE, "ptxas.log"), "w") as fh:
        fh.write("\n".join(log))
    if verbose:
        sys.stderr.write("\n".join(log))
    os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
