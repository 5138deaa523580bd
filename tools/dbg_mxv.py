"""Debug helper: run one pp_mxv combination (used under compute-sanitizer)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import synth, oracle
import paper_1804_03327_b200 as pp
from test_gpu_mxv import dev_vec, read_vec, expected

ctx = pp.Context(0)
g = synth.random_graph(1999, 12000, seed=4, symmetrize=False)
gT = synth.transpose(g)
G = pp.Graph.from_csr(ctx, g, gT, validate=True)
n = g.n
rng = np.random.default_rng(3)
u = (rng.random(n) < 0.3).astype(np.uint8)
w_in = np.zeros(n, np.uint8)
for ufmt in (pp.PP_VEC_BITMAP, pp.PP_VEC_LIST):
    for direction in (pp.PP_DIR_PULL, pp.PP_DIR_PUSH):
        uvec, ut = dev_vec(u, ufmt)
        wvec, wt = dev_vec(w_in, pp.PP_VEC_BITMAP)
        try:
            pp.mxv(G, wvec, uvec, direction=direction)
            got = read_vec(wvec, wt, n)
            print(ufmt, direction, "ok" if np.array_equal(got, expected(g, gT, u, None, 0, 0, 1, w_in, 1)) else "MISMATCH", flush=True)
        except Exception as e:
            print(ufmt, direction, "ERR", e, flush=True)
            raise
