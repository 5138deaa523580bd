"""Build libpushpull.so (CUDA for sm_100a + the C ABI) in-tree with nvcc."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "libpushpull.so")
SOURCES = ["bfs.cu", "mxv.cu", "graph.cu", "relabel.cu", "dist.cu", "sssp.cu", "capi.cpp"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
         "-Xcompiler", "-fPIC,-O3", "-shared", "-cudart", "static", "-I", os.path.join(ROOT, "include"),
         "-I", CSRC]


def needs_build():
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "pushpull.h")]
    return any(os.path.getmtime(p) > t for p in deps)


def build(force=False, verbose=False):
    """Compile every source to an object in parallel, then link the shared library."""
    if not force and not needs_build():
        return SO
    import concurrent.futures as cf
    tmp = SO + f".tmp{os.getpid()}"
    extra = [f"-D{k}={os.environ[k]}" for k in ("PP_BFS_BLOCK", "PP_SUM_WORDS", "PP_PULL_WORDS", "PP_PULL_KC", "PP_SOLO_EDGES", "PP_LOWLAT_EDGES", "PP_NARROW_MAX_EDGES", "PP_NARROW_MAX_DEG", "PP_VREC", "PP_INIT_VEC", "PP_STREAM_U", "PP_SSSP_G", "PP_SSSP_HEAVY") if os.environ.get(k)]
    extra += ["-DPP_IDX_NOALLOC"] if os.environ.get("PP_IDX_NOALLOC") else []
    extra += [f"-D{k}" for k in ("PP_KO_DEPTH", "PP_KO_PROBE", "PP_KO_RESID") if os.environ.get(k)]
    extra += [f"-D{k}={os.environ[k]}" for k in ("PP_FAST_NTH", "PP_PUSH_KU", "PP_STEAL",
                                                   "PP_LOWLAT_VREC", "PP_PF_ROWS",
                                                   "PP_SUM_RESID", "PP_DENSE", "PP_DENSE_R",
                                                   "PP_DENSE_MIN8", "PP_DENSE_IW",
                                                   "PP_CHUNK", "PP_HEAVY", "PP_RQ_EXTRA", "PP_DENSE_DIST", "PP_BAR_ACQREL", "PP_BAR_SLEEP")
              if os.environ.get(k)]
    odir = os.path.join(HERE, "build")
    os.makedirs(odir, exist_ok=True)
    cflags = [f for f in FLAGS if f != "-shared"]

    def comp(src):
        obj = os.path.join(odir, src + f".{os.getpid()}.o")
        cmd = [NVCC] + cflags + extra + (["-Xptxas", "-v"] if verbose else []) + \
            ["-c", os.path.join(CSRC, src), "-o", obj]
        subprocess.check_call(cmd)
        return obj

    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(comp, SOURCES))
    subprocess.check_call([NVCC] + FLAGS + objs + ["-ldl", "-o", tmp])
    for o in objs:
        os.unlink(o)
    os.replace(tmp, SO)
    return SO


if __name__ == "__main__":
    print(build(force=True, verbose="-v" in sys.argv))
