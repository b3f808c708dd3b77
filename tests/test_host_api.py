"""CPU-only tests of the drop-in boundary: registry/dispatch contract
(mirrors pkg/tests/test_dispatch.py), tuning validation, host containers
(mirrors pkg/tests/test_sparse.py validation cases), and the C-ABI library
(loads, exports every symbol include/wk_sparse.h declares; no compute)."""

import os
import re
import subprocess

import numpy as np
import pytest

import paper_2006_14290_b200 as wk
from paper_2006_14290_b200 import _lib
from paper_2006_14290_b200.dispatch import EXEC_B200, EXEC_REFERENCE, Operation

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class TestLibrary:
    def test_header_symbols_exported(self):
        header = open(os.path.join(ROOT, "include", "wk_sparse.h")).read()
        declared = set(re.findall(r"^(?:int|int64_t|const char\*)\s+(wk_[a-z0-9_]+)\s*\(", header, re.M))
        assert declared, "no declarations found"
        assert declared == set(_lib.EXPORTED), declared ^ set(_lib.EXPORTED)
        out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True,
                             check=True).stdout
        exported = {line.split()[-1] for line in out.splitlines() if line.split()[-1].startswith("wk_")}
        assert declared <= exported, declared - exported

    def test_library_loads_and_reports(self):
        L = _lib.load()
        assert L.wk_version() >= 1
        assert L.wk_reduce_workspace_bytes() > 0
        assert L.wk_csr_plan_chunks(0) == 1 and L.wk_csr_plan_chunks(257) == 2
        assert L.wk_cg_workspace_bytes(1000) > 3 * 8000

    def test_sm100a_cubin_only(self):
        out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
        assert "sm_100a" in out

    def test_status_mapping(self):
        with pytest.raises(wk.BreakdownError):
            _lib.check(_lib.WK_ERR_BREAKDOWN)
        with pytest.raises(wk.DimensionMismatch):
            _lib.check(_lib.WK_ERR_DIMENSION)
        with pytest.raises(wk.InvalidSliceSize):
            _lib.check(_lib.WK_ERR_SLICE)
        with pytest.raises(ValueError):
            _lib.check(_lib.WK_ERR_INVALID)
        with pytest.raises(wk.DeviceError):
            _lib.check(2)


class TestExecutor:
    def test_factory_kinds(self):
        assert wk.make_executor("b200").kind == EXEC_B200
        assert wk.make_executor("ref").kind == EXEC_REFERENCE
        assert wk.make_executor("b200").warp_size == 32
        with pytest.raises(ValueError):
            wk.make_executor("warp128")

    def test_custom_tuning(self):
        ex = wk.make_executor("b200", tuning={"block_size": 128, "subwarps_per_block": 32, "csr_subwarp_size": 4})
        assert ex.config.tuning["csr_subwarp_size"] == 4
        assert ex.config.tuning["csr_strategy"] == "auto"

    def test_tuning_validation(self):
        with pytest.raises(ValueError):
            wk.B200Config({"block_size": 100})
        with pytest.raises(ValueError):
            wk.B200Config({"block_size": 2048})
        with pytest.raises(ValueError):
            wk.B200Config({"csr_subwarp_size": 64})
        with pytest.raises(ValueError):
            wk.B200Config({"csr_strategy": "balanced"})
        with pytest.raises(ValueError):
            wk.make_executor("ref", tuning={"block_size": 256})


class TestRegistry:
    def test_known_operations_present(self):
        names = wk.registered_operations()
        for expected in ("spmv_coo", "spmv_csr", "spmv_sellp", "spmv_ell", "spmv_hybrid", "cg", "bicgstab",
                         "gmres", "dot", "norm2", "axpy", "coo_to_csr", "coo_to_sellp", "csr_to_ell",
                         "csr_to_sellp", "csr_to_hybrid"):
            assert expected in names

    def test_every_operation_has_b200_impl(self):
        for name in wk.registered_operations():
            assert wk.get_operation(name).impls.get(EXEC_B200) is not None

    def test_b200_impl_required(self):
        with pytest.raises(ValueError):
            Operation("broken", {EXEC_REFERENCE: lambda exec: None})
        with pytest.raises(ValueError):
            Operation("broken", {EXEC_B200: lambda e: 0, "sim-warp32": lambda e: 0})

    def test_missing_backend_raises(self):
        op = Operation("b200_only", {EXEC_B200: lambda exec: 1.0})
        assert wk.dispatch(op, wk.make_executor("b200")) == 1.0
        with pytest.raises(wk.NotImplementedForBackend):
            wk.dispatch(op, wk.make_executor("ref"))

    def test_explicit_not_implemented_marker(self):
        op = Operation("marked", {EXEC_B200: lambda exec: 0, EXEC_REFERENCE: None})
        with pytest.raises(wk.NotImplementedForBackend):
            wk.dispatch(op, wk.make_executor("ref"))

    def test_unregistered_name(self):
        with pytest.raises(KeyError):
            wk.dispatch("no_such_op", wk.make_executor("b200"))

    def test_counters_reset_and_accumulate(self):
        def impl(exec):
            exec.counters.lane_steps += 5
            return exec.counters.lane_steps

        op = Operation("count", {EXEC_B200: impl})
        ex = wk.make_executor("b200")
        assert wk.dispatch(op, ex) == 5
        assert wk.dispatch(op, ex) == 5
        ex.accumulate = True
        assert wk.dispatch(op, ex) == 10
        snap = wk.instrumentation_report(ex)
        snap.lane_steps = 999
        assert ex.counters.lane_steps == 10

    def test_reference_slot_can_be_registered_by_callers(self):
        from oracle import sparse_ref

        op = Operation("spmv_with_ref", {EXEC_B200: lambda e, m, x: None,
                                         EXEC_REFERENCE: lambda e, m, x: sparse_ref.spmv(m, x)})
        m = wk.CsrMatrix(2, 2, [0, 1, 2], [0, 1], [2.0, 3.0])
        assert np.array_equal(wk.dispatch(op, wk.make_executor("ref"), m, np.ones(2)), [2.0, 3.0])


class TestHostContainers:
    def test_coo_validation(self):
        with pytest.raises(ValueError):
            wk.CooMatrix(2, 2, [0, 3], [0, 0], [1.0, 1.0])
        with pytest.raises(ValueError):
            wk.CooMatrix(2, 2, [1, 0], [0, 0], [1.0, 1.0])
        with pytest.raises(ValueError):
            wk.CooMatrix(2, 2, [0, 0], [1, 1], [1.0, 1.0])

    def test_csr_validation(self):
        with pytest.raises(ValueError):
            wk.CsrMatrix(2, 2, [0, 1], [0], [1.0])
        with pytest.raises(ValueError):
            wk.CsrMatrix(2, 2, [0, 2, 2], [1, 0], [1.0, 1.0])  # decreasing columns
        with pytest.raises(ValueError):
            wk.CsrMatrix(2, 2, [0, 1, 2], [0, 2], [1.0, 1.0])  # out of bounds
        m = wk.CsrMatrix(3, 3, [0, 2, 3, 5], [0, 2, 1, 0, 2], [1.0, 2.0, 3.0, 4.0, 5.0])
        assert np.array_equal(m.to_dense(), [[1, 0, 2], [0, 3, 0], [4, 0, 5]])

    def test_sellp_validation_and_dense(self):
        with pytest.raises(wk.InvalidSliceSize):
            wk.SellpMatrix(3, 3, 3, [0, 2], np.zeros(6), np.zeros(6), [1, 1, 1])
        sp = wk.SellpMatrix(3, 3, 2, [0, 2, 4], [0, 1, 2, 0, 0, 0, 2, 0], [1.0, 3.0, 2.0, 0.0, 4.0, 0.0, 5.0, 0.0],
                            [2, 1, 2])
        assert np.array_equal(sp.to_dense(), [[1, 0, 2], [0, 3, 0], [4, 0, 5]])
        assert sp.nslices == 2 and sp.slice_width(1) == 2 and sp.nnz == 5

    def test_ell_hybrid_validation(self):
        with pytest.raises(ValueError):
            wk.EllMatrix(3, 3, 2, 2, np.zeros(4), np.zeros(4), [0, 0, 0])  # stride < nrows
        ell = wk.EllMatrix(2, 2, 1, 2, [1, 0], [5.0, 6.0], [1, 1])
        coo = wk.CooMatrix(2, 2, [0], [0], [1.0])
        h = wk.HybridMatrix(2, 2, ell, coo)
        assert np.array_equal(h.to_dense(), [[1, 5], [6, 0]])
        assert np.array_equal(h.row_nnz(), [2, 1])

    def test_accepts_reference_field_layout(self):
        from oracle import sparse_ref

        ns = sparse_ref.csr_to_sellp(sparse_ref.coo_to_csr(sparse_ref.coo_from_entries(
            3, 3, [0, 0, 1, 2, 2], [0, 2, 1, 0, 2], [1.0, 2.0, 3.0, 4.0, 5.0])), 2)
        sp = wk.SellpMatrix(ns.nrows, ns.ncols, ns.slice_size, ns.slice_sets, ns.col_idx, ns.values, ns.row_lengths)
        assert sp.slice_sets.tolist() == [0, 2, 4]


class TestStoppingCriteria:
    def test_criteria_validation(self):
        with pytest.raises(ValueError):
            wk.ResidualNorm(0.0)
        with pytest.raises(ValueError):
            wk.ResidualNorm(1e-8, baseline="other")
        f = wk.Cg([wk.Iteration(10), wk.ResidualNorm(1e-8)])
        assert f.kind == "cg" and len(f.criteria) == 2
        assert wk.Gmres(restart=20).restart == 20
