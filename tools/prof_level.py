"""Run ONE BFS level alone in its own launch (pp_bfs_debug_level) so ncu can capture it:
  ncu --set full -k regex:bfs_persistent --launch-skip S --launch-count 1 \
      python tools/prof_level.py [CONFIG] [LEVEL|pull|push] [SOURCE_INDEX]
The first call is a warm-up (2 launches), the second call's second launch is the level alone
(--launch-skip 4: launch 0 is the stats BFS).  Prints the level's direction, frontier and candidate counts."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
import paper_1804_03327_b200 as pp  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
which = sys.argv[2] if len(sys.argv) > 2 else "pull"
si = int(sys.argv[3]) if len(sys.argv) > 3 else 5
g = synth.make(cfg)
ctx = pp.Context(0)
G = pp.Graph.from_csr(ctx, g, relabel=True)
s = int(synth.sources(g, 64, seed=2)[si])
d = torch.zeros(g.n, dtype=torch.int32, device="cuda")
st = pp.bfs(G, s, d, stats_capacity=4096)
dirs = list(st["dir"])
if which in ("pull", "push"):
    want = 1 if which == "pull" else 0
    cand = [k for k in range(len(dirs)) if dirs[k] == want]
    # the heaviest: the pull with the most candidates is the first pull; the push with the largest
    # new frontier for push
    level = (cand[0] if want == 1 else max(cand, key=lambda k: st["c"][k])) + 1
else:
    level = int(which)
print(f"{cfg} source {s}: dirs {''.join('HL'[x] for x in dirs)}; profiling level {level} "
      f"({'HL'[dirs[level - 1]]}, discovers {st['c'][level - 1]})", flush=True)
for _ in range(2):
    pp.pp_bfs_debug_level(G.handle, s, level, d.data_ptr())
torch.cuda.synchronize()
