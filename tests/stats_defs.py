"""Expected pp_bfs_stats.cand / reached_nnz, counted from their definitions on oracle depths."""
import numpy as np


def expected_cand(g, gT, ed, dirs, no_mask=False):
    """pp_bfs_stats.cand from its definition: a pull level k computes the rows that are
    neither isolated nor visited before it (depth 0 or > k; P:270 masking), every
    non-isolated row without masking; a push level k expands the frontier {depth == k}."""
    noniso = (np.diff(g.off) > 0) | (np.diff(gT.off) > 0)
    out = []
    for k, dr in enumerate(dirs, start=1):
        if dr == 1:
            out.append(int(noniso.sum()) if no_mask else int((noniso & ((ed == 0) | (ed > k))).sum()))
        else:
            out.append(int((ed == k).sum()))
    return np.array(out, np.int64)


def check_cand(g, gT, ed, st, no_mask=False):
    assert np.array_equal(st["cand"], expected_cand(g, gT, ed, st["dir"], no_mask)), st["cand"]
    assert st["reached_nnz"] == int(np.diff(gT.off)[ed > 0].sum())
