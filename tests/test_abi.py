"""C-ABI library checks that need no GPU: it loads, exports every symbol that
include/pushpull.h declares, and fails loudly (no CPU fallback) without a device."""
import ctypes
import re
import subprocess

import pytest
import torch

import paper_1804_03327_b200 as pp


def test_exports_every_header_symbol():
    declared = pp.header_functions()
    assert len(declared) >= 12
    out = subprocess.run(["nm", "-D", "--defined-only", pp.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (pp_\w+)$", out, re.M))
    missing = [f for f in declared if f not in exported]
    assert not missing, missing
    lib = ctypes.CDLL(pp.LIB_PATH)
    for f in declared:
        assert hasattr(lib, f)
    assert set(pp.EXPORTED) == set(declared)


def test_library_is_sm100a_native():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", pp.LIB_PATH],
                         capture_output=True, text=True, check=True).stdout
    assert "sm_100a" in out


def test_defaults_and_version():
    assert "sm_100a" in pp.pp_version()
    d = pp.pp_descriptor_default()
    assert d.replace == 1 and d.early_exit == 1 and d.transpose == 1 and abs(d.switchpoint - 0.01) < 1e-15
    assert d.prev_nnz == -1 and not d.mask
    o = pp.pp_bfs_options_default()
    assert o.heuristic == pp.PP_HEUR_EDGES and o.mode == pp.PP_MODE_DO and o.toggles == 0


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure path")
def test_no_gpu_fails_loudly():
    with pytest.raises(pp.PPError) as e:
        pp.pp_ctx_create(0, 0)
    assert e.value.status == pp.PP_ERR_CUDA
    assert "no CPU fallback" in str(e.value)


def test_null_arguments_rejected():
    with pytest.raises(pp.PPError) as e:
        pp.pp_graph_free(None)
    assert e.value.status == pp.PP_ERR_ARG
    with pytest.raises(pp.PPError) as e:
        pp.pp_ctx_destroy(None)
    assert e.value.status == pp.PP_ERR_ARG
