"""The reference's per-layer cost model (config.h:40-66,
config.cc:23-118) restated in paper_2412_12488_b200/cost_model.py, checked
against the compiled reference: DefaultCostModel from the shipped anchors,
fits of random anchor sets, the degenerate / too-few-anchor errors and the
piecewise definitions (X(n <= 0) = 0, empty decode batch = 0)."""
import ctypes as C

import numpy as np
import pytest

from paper_2412_12488_b200 import ErrorCode, SplitserveError
from paper_2412_12488_b200.cost_model import (DEFAULT_PREFILL_ANCHORS, DEFAULT_TRANSFER_ANCHORS,
                                              CostModel, default_cost_model, fit_cost_model)


def _ref(ref_lib):
    lib = C.CDLL(ref_lib)
    lib.ssref_default_cost_model.argtypes = [C.POINTER(C.c_double)]
    lib.ssref_fit_cost_model.argtypes = [C.POINTER(C.c_double), C.c_int32, C.POINTER(C.c_double),
                                         C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_double)]
    return lib


def _fields(m: CostModel):
    return [m.alpha, m.beta, m.gamma, m.delta, m.c0, m.c1]


def _ref_fit(lib, prefill, transfer):
    p = (C.c_double * (3 * len(prefill)))(*[float(x) for a in prefill for x in a])
    t = (C.c_double * (2 * len(transfer)))(*[float(x) for a in transfer for x in a])
    out = (C.c_double * 6)()
    err = C.c_double()
    st = lib.ssref_fit_cost_model(p, len(prefill), t, len(transfer), out, C.byref(err))
    return st, list(out), err.value


def test_default_cost_model_matches_reference(ref_lib):
    lib = _ref(ref_lib)
    out = (C.c_double * 6)()
    assert lib.ssref_default_cost_model(out) == 0
    ours = _fields(default_cost_model())
    assert ours == list(out)  # same arithmetic, same order: bit-identical
    # the fitted transfer line reproduces the paper's anchors to within 1%
    m = default_cost_model()
    for n, ms in DEFAULT_TRANSFER_ANCHORS:
        assert abs(m.transfer_layer_ms(n) - ms) / ms < 0.01
    for u, t, ms in DEFAULT_PREFILL_ANCHORS:
        assert abs(m.prefill_layer_ms(u, t) - ms) / ms < 0.02


def test_random_fits_match_reference(ref_lib):
    lib = _ref(ref_lib)
    rng = np.random.default_rng(7)
    for _ in range(50):
        n_p, n_t = int(rng.integers(2, 6)), int(rng.integers(2, 6))
        prefill = [(int(rng.integers(1, 4000)), int(rng.integers(1, 32768)),
                    float(rng.uniform(0.01, 10))) for _ in range(n_p)]
        transfer = [(int(rng.integers(1, 32768)), float(rng.uniform(0.001, 5))) for _ in range(n_t)]
        st, want, want_err = _ref_fit(lib, prefill, transfer)
        if st != 0:
            with pytest.raises(SplitserveError):
                fit_cost_model(prefill, transfer)
            continue
        rep = fit_cost_model(prefill, transfer)
        assert _fields(rep.model) == want
        assert rep.max_rel_err == want_err


def test_fit_errors_match_reference(ref_lib):
    lib = _ref(ref_lib)
    cases = [
        ([(500, 1000, 1.0)], [(1000, 0.2), (2000, 0.4)]),          # one prefill anchor
        ([(500, 1000, 1.0), (500, 2000, 1.1)], [(1000, 0.2)]),      # one transfer anchor
        ([(500, 1000, 1.0), (500, 2000, 1.1)], [(1000, 0.2), (1000, 0.3)]),  # degenerate
    ]
    for prefill, transfer in cases:
        st, _, _ = _ref_fit(lib, prefill, transfer)
        assert st == 1 + ErrorCode.InvalidArgument
        with pytest.raises(SplitserveError) as ei:
            fit_cost_model(prefill, transfer)
        assert ei.value.code == ErrorCode.InvalidArgument


def test_piecewise_definitions():
    m = CostModel(alpha=1e-3, beta=2e-7, gamma=1.6e-4, delta=0.03)
    assert m.transfer_layer_ms(0) == 0.0 and m.transfer_layer_ms(-5) == 0.0
    assert m.transfer_layer_ms(1000) == pytest.approx(0.19)
    assert m.decode_layer_ms([]) == 0.0
    assert m.decode_layer_ms([100, 300]) == pytest.approx(0.05 + 2e-5 * 400)
    assert m.prefill_layer_ms(500, 1000) == pytest.approx(0.5 + 0.1)
    m.validate()
    with pytest.raises(SplitserveError) as ei:
        CostModel(gamma=-1.0).validate()
    assert ei.value.code == ErrorCode.InvalidArgument
