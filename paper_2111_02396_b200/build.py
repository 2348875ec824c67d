"""Build libqtraj.so (sm_100a) in-tree with nvcc; parallel per-file compile."""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.environ.get("QT_LIB_OUT", os.path.join(HERE, "libqtraj.so"))
OBJ = os.path.join(HERE, "build_obj" + os.environ.get("QT_OBJ_SUFFIX", ""))
SOURCES = ["tile_pass_r4.cu", "tile_pass_r5.cu", "tile_pass_r6.cu", "tile_pass_tc.cu", "tile_pass_tcw.cu",
           "tile_pass_v2.cu", "tile_pass_v3.cu", "gate_stream.cu", "tile_pass_r5s.cu", "tile_pass_r6s_a.cu", "tile_pass_r6s_b.cu", "kernels.cu",
           "circuit.cpp", "planner.cpp", "runtime.cpp", "dist_host.cpp"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2"]
# experiment builds: QT_EXTRA_FLAGS="-DQT_TC_EXP=1" QT_LIB_OUT=... QT_OBJ_SUFFIX=_exp
FLAGS += os.environ.get("QT_EXTRA_FLAGS", "").split()


def _deps():
    return [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + \
        [os.path.join(HERE, "..", "include", "qtraj.h")]


def needs_build():
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    return any(os.path.getmtime(p) > t for p in _deps())


def build(force=False, verbose=False):
    if not force and not needs_build():
        return OUT
    os.makedirs(OBJ, exist_ok=True)

    def compile_one(src):
        obj = os.path.join(OBJ, src + ".o")
        cmd = [NVCC] + ARCH + FLAGS + ["-c", os.path.join(CSRC, src), "-o", obj]
        if src.endswith(".cu"):
            cmd += ["-Xptxas", "-v"] if verbose else []
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
        return obj

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    cmd = [NVCC] + ARCH + ["-shared", "-o", OUT + ".tmp"] + objs + ["-lpthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(OUT)
