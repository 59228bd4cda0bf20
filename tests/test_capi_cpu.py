"""CPU-side checks of the product library: it loads, exports every symbol the
C-ABI header declares, and its host logic (LIFO allocator mirror, config
validation / error mapping, technique names) matches the reference."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_2407_20272_b200 import exitlab as X
from paper_2407_20272_b200.build import LIB

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "exitlab_b200.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(el_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    assert os.path.exists(LIB), "build() first"
    lib = ctypes.CDLL(LIB)
    syms = declared_symbols()
    assert len(syms) >= 25
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert lib.el_version() == 1


def test_kv_block_trace_host_mirror_matches_reference_golden(golden):
    for c in golden("kv_block_traces.json"):
        tab, nf = X.kv_block_trace(c["L"], c["pool"], c["cap"], c["ops"], c["caps"], c["n_ids"], c["bpl_max"])
        assert nf == c["free"]
        assert tab.tolist() == c["tables"]


def test_kv_block_trace_lifo_examples():
    # fresh pool pops 0,1,2,... layer-major (kv_cache.cpp:53-55, 96-103)
    tab, nf = X.kv_block_trace(3, 64, 16, [1], [20], 1, 4)
    assert tab[0, :, :2].tolist() == [[0, 1], [2, 3], [4, 5]] and nf == 58
    # release pushes in table order, the next allocation gets them reversed
    tab, nf = X.kv_block_trace(3, 64, 16, [1, -1, 2], [16, 0, 16], 2, 2)
    assert tab[1, :, 0].tolist() == [2, 1, 0]
    # KvOutOfMemory defers without leaking (test_kv_cache.cpp:29-33)
    tab, nf = X.kv_block_trace(8, 7, 16, [1], [1], 1, 1)
    assert nf == 7 and tab[0, 0, 0] == -1
    with pytest.raises(ValueError):
        X.kv_block_trace(2, 16, 4, [-1], [0], 1, 1)  # release of an unknown id


@pytest.mark.parametrize("patch,msg", [
    (dict(max_batch=0), "max_batch"),
    (dict(technique=X.ExitTechnique.always_at(9)), "always_at"),
    (dict(schedule=X.ThresholdSchedule(0.5, 0.0, 0.0)), "gamma"),
    (dict(schedule=X.ThresholdSchedule(0.5, 1.0, 0.6)), "lambda_min"),
    (dict(model=X.ModelConfig(1, 8, 16, 0)), "n_layers"),
    (dict(eos_token=16), "eos_token"),
])
def test_config_validation_raises_invalid_argument(patch, msg):
    # mirrors test_engine.cpp:326-338 / test_model.cpp:28-32; validation precedes any device call
    base = dict(model=X.ModelConfig(3, 8, 16, 11), technique=X.ExitTechnique.never(), max_batch=4, pool_blocks=256,
                block_capacity=4)
    base.update(patch)
    with pytest.raises(ValueError, match=msg):
        X.Engine(X.EngineConfig(**base))


def test_technique_names_round_trip():
    for name in ["softmax", "state", "classifier", "never", "always-at=4"]:
        assert X.technique_from_name(name).name == name
    for bad in ["bogus", "always-at=x", "always-at=0"]:
        with pytest.raises(ValueError):
            X.technique_from_name(bad)


def test_workload_flat_round_trip():
    w = X.Workload([X.Request(0.0, [1, 2, 3], 4), X.Request(0.5, [7], 2)])
    flat = w.flat()
    back = X.Workload.from_flat(*flat)
    assert back == w


def test_create_sized_rejects_unknown_nonzero_fields():
    """el_engine_create_sized: a caller's struct longer than the library's may only carry zeros
    past it (checked before any device work, so this runs without a GPU)."""
    import ctypes as C
    from paper_2407_20272_b200 import exitlab as X
    lib = X.lib()
    n = C.sizeof(X._CConfig)
    buf = (C.c_ubyte * (n + 8))()
    buf[n + 3] = 1
    h = C.c_void_p()
    rc = lib.el_engine_create_sized(C.cast(buf, C.c_void_p), n + 8, C.byref(h))
    assert rc == 1 and not h.value  # EL_INVALID_ARGUMENT
    assert b"unknown non-zero field" in lib.el_last_error()
