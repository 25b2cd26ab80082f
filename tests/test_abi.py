"""The C-ABI boundary (include/ds_blstm.h): libds.so loads on any host and
exports every declared entry point; host-side validation errors come back as
the reference's exception types without touching a GPU."""

import ctypes
import os
import re

import pytest

from paper_1904_04956_b200 import _lib

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "ds_blstm.h")


def _declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|int32_t|int64_t|const char\*)\s+(ds_\w+)\s*\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    names = _declared()
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) <= set(_lib.SIGNATURES), set(names) - set(_lib.SIGNATURES)


def test_param_dim_and_config_validation():
    lib = _lib.load()
    cfg = _lib.DsCfg(6, 260, 256, 32000, 21, 256)
    assert lib.ds_blstm_param_dim(ctypes.byref(cfg)) == 43_130_368
    bad = _lib.DsCfg(6, 300, 256, 32000, 21, 256)  # input_dim > 272
    assert lib.ds_blstm_param_dim(ctypes.byref(bad)) == -1
    h = ctypes.c_void_p()
    rc = lib.ds_blstm_create(ctypes.byref(bad), 0, ctypes.byref(h))
    with pytest.raises(ValueError, match="input_dim"):
        _lib.check(rc)


def test_host_side_argument_errors():
    lib = _lib.load()
    with pytest.raises(ValueError):
        _lib.check(lib.ds_adpsgd_mix(None, None, 10, None))
    with pytest.raises(ValueError, match="learning rate"):
        _lib.check(lib.ds_sgd_momentum(1, 1, 1, -0.1, 0.9, 10, None, None, None))
    with pytest.raises(ValueError, match="rank"):
        _lib.check(lib.ds_group_reduce(2, 5, None, (ctypes.c_void_p * 2)(1, 1), None, None, 10, 2, 0.1, 0.9, 0, 0.0,
                                       None))


def test_objective_config_matches_c_layout():
    from paper_1904_04956_b200.blstm import BlstmObjective

    lib = _lib.load()
    for obj in (BlstmObjective(), BlstmObjective(layers=2, classes=512, frames=5), BlstmObjective(layers=1, bottleneck=64)):
        cfg = obj.cfg(8)
        assert lib.ds_blstm_param_dim(ctypes.byref(cfg)) == obj.param_dim
