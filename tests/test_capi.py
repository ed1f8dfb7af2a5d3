"""C-ABI library checks that need no GPU (-m "not gpu").

* libphub.so loads and exports every entry point include/phub.h declares;
* the host-side planner (phub_plan_chunks) reproduces the oracle's chunk
  table and owner tables exactly (byte-equal canonical text);
* validation happens on the host before any CUDA call.
"""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "phub.h")


def _declared():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(phub_[a-z_]+)\s*\(", txt)))


def test_library_loads_and_exports_every_declared_symbol():
    from paper_1805_07891_b200 import capi
    lib = capi.raw_lib()
    declared = _declared()
    assert "phub_init" in declared and "phub_aggregate_optimize" in declared
    for name in declared:
        assert hasattr(lib, name), name
    # the binding covers exactly the declared surface
    assert sorted(capi.EXPORTS) == declared
    out = subprocess.run(["nm", "-D", "--defined-only", capi.LIB_PATH], capture_output=True,
                         text=True).stdout
    exported = set(re.findall(r" T (phub_\w+)", out))
    assert set(declared) <= exported


def test_status_strings_and_defaults():
    from paper_1805_07891_b200 import capi
    assert capi.phub_status_string(0) == "PHUB_OK"
    assert capi.phub_status_string(capi.PHUB_ERR_DUPLICATE_PUSH) == "PHUB_ERR_DUPLICATE_PUSH"
    assert capi.phub_status_string(999) == "PHUB_ERR_UNKNOWN"
    cfg = capi.phub_config_default()
    assert cfg.chunk_size_bytes == 32768          # P:697 default 32KB
    assert cfg.num_owners == 1 and cfg.owner_policy == capi.PHUB_OWNER_CONTIG
    assert abs(cfg.lr - 0.1) < 1e-7 and abs(cfg.momentum - 0.9) < 1e-7


def _init_status(**kw):
    from paper_1805_07891_b200 import capi
    sizes = kw.pop("sizes", [10, 20])
    arr = (C.c_uint64 * max(len(sizes), 1))(*sizes)
    cfg = capi.phub_config_default()
    cfg.key_num_elements = arr
    cfg.num_keys = len(sizes)
    cfg.num_workers = 2
    for k, v in kw.items():
        setattr(cfg, k, v)
    ctx = capi.phub_ctx()
    return capi.raw_lib().phub_init(C.byref(cfg), C.byref(ctx)), ctx


@pytest.mark.parametrize("kw,status", [
    (dict(sizes=[]), "PHUB_ERR_INVALID_MANIFEST"),
    (dict(sizes=[4, 0]), "PHUB_ERR_INVALID_MANIFEST"),
    (dict(chunk_size_bytes=6), "PHUB_ERR_INVALID_CHUNK_SIZE"),
    (dict(num_workers=0), "PHUB_ERR_INVALID_ARGUMENT"),
    (dict(momentum=1.0), "PHUB_ERR_INVALID_ARGUMENT"),
    (dict(lr=float("nan")), "PHUB_ERR_INVALID_ARGUMENT"),
    (dict(num_owners=2, owner_rank=2), "PHUB_ERR_INVALID_ARGUMENT"),
    (dict(owner_policy=7), "PHUB_ERR_INVALID_ARGUMENT"),
])
def test_init_validation_is_host_side(kw, status):
    from paper_1805_07891_b200 import capi
    st, ctx = _init_status(**kw)
    assert capi.STATUS_NAMES[st] == status
    assert not ctx.value
    assert capi.phub_last_error(None)          # thread-local init error detail


@pytest.mark.parametrize("name", ["tiny", "resnet50", "alexnet", "vgg19", "resnet269"])
@pytest.mark.parametrize("G", [1, 2, 4, 8])
@pytest.mark.parametrize("policy", ["lpt", "contig"])
def test_plan_matches_oracle(name, G, policy):
    import oracle
    from paper_1805_07891_b200 import capi
    from workloads import manifest
    m = manifest(name)
    pol = capi.PHUB_OWNER_LPT if policy == "lpt" else capi.PHUB_OWNER_CONTIG
    arr, n = capi.phub_plan_chunks(m, 32768, G, pol)
    lib = np.ctypeslib.as_array(arr)[:n]
    ref = oracle.chunk_plan(m, 32768)
    own = (oracle.owners_lpt if policy == "lpt" else oracle.owners_contig)(ref["length"], G)
    if G == 1:
        own = np.zeros_like(own)
    assert oracle.canonical_text(
        {f: np.array(lib[f]) for f in ("vkey_id", "key_id", "offset", "length")},
        np.array(lib["owner"])) == oracle.canonical_text(ref, own)


@pytest.mark.parametrize("cb", [4, 12, 4096, 8192, 16384, 65536, 131072, 262144, 524288,
                                1048576])
def test_plan_sweep_matches_oracle(cb):
    import oracle
    from paper_1805_07891_b200 import capi
    from workloads import manifest
    m = manifest("resnet269") if cb >= 4096 else [3, 3, 100, 7, 4097]
    arr, n = capi.phub_plan_chunks(m, cb, 4, capi.PHUB_OWNER_LPT)
    lib = np.ctypeslib.as_array(arr)[:n]
    ref = oracle.chunk_plan(m, cb)
    assert n == len(ref["length"])
    for f in ("vkey_id", "key_id", "offset", "length"):
        assert np.array_equal(np.array(lib[f]).astype(np.uint64), ref[f].astype(np.uint64))
    assert np.array_equal(np.array(lib["owner"]), oracle.owners_lpt(ref["length"], 4))


def test_c_example_builds_against_the_abi():
    """A plain-C program (no Python, no torch) compiles and links against
    include/phub.h + libphub.so; its run is a GPU test."""
    import runpy
    b = runpy.run_path(os.path.join(ROOT, "paper_1805_07891_b200", "build.py"))
    exe = b["build_example"]()
    assert os.path.exists(exe)
    out = subprocess.run(["ldd", exe], capture_output=True, text=True).stdout
    assert "libphub.so" in out


def test_struct_layouts_match_the_header(tmp_path):
    """The ctypes mirrors of the ABI structs have the C compiler's sizes and
    field offsets (a drifted mirror would pass garbage across the boundary)."""
    from paper_1805_07891_b200 import capi
    structs = {"phub_config": capi.phub_config, "phub_chunk": capi.phub_chunk,
               "phub_sync": capi.phub_sync, "phub_hier": capi.phub_hier}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "phub.h"', "int main(void){"]
    for name, cls in structs.items():
        lines.append(f'printf("{name} %zu\\n", sizeof({name}));')
        for fname, _t in cls._fields_:
            lines.append(f'printf("{name}.{fname} %zu\\n", offsetof({name}, {fname}));')
    lines.append("return 0;}")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), "-o", str(exe), str(src)])
    got = dict(ln.split() for ln in subprocess.check_output([str(exe)], text=True).splitlines())
    for name, cls in structs.items():
        assert int(got[name]) == C.sizeof(cls), name
        for fname, _t in cls._fields_:
            assert int(got[f"{name}.{fname}"]) == getattr(cls, fname).offset, f"{name}.{fname}"
