"""The reference's zero-atomics contract for SELL-P (kernels.py:146-149,
test_acceptance.py:216-229) checked on the compiled sm_100a code instead of
a simulator counter: the SASS of the default SELL-P, ELL and CSR-rowblock SpMV
kernels holds no atomic / reduction instruction (ATOM, ATOMG, RED, REDG),
while the COO kernel (kernels.py:229-253 semantics: run-head atomics) does.
The same listing proves the TMA path (UBLKCP = cp.async.bulk) of the SELL-P
kernel. CPU-only: cuobjdump on the built library."""

import os
import re
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2006_14290_b200", "_lib", "libwk_sparse.so")

ATOMIC = re.compile(r"\b(ATOM|ATOMG|ATOMS|RED|REDG|REDUX)\b")


@pytest.fixture(scope="module")
def sass():
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(LIB) or not os.path.exists(tool):
        pytest.skip("library or cuobjdump missing")
    out = subprocess.run([tool, "-sass", LIB], check=True, capture_output=True, text=True).stdout
    funcs, name, body = {}, None, []
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            if name:
                funcs[name] = "\n".join(body)
            name, body = m.group(1), []
        elif name:
            body.append(line)
    if name:
        funcs[name] = "\n".join(body)
    return funcs


def _pick(funcs, *parts):
    hits = [k for k in funcs if all(p in k for p in parts)]
    assert hits, parts
    return hits


def test_sellp_spmv_has_no_atomics_and_uses_tma(sass):
    # both SpMV configurations (wide SellpTmaCfg<4,3,16,1>, narrow <2,5,24,1>), kDot = kCoh = false, kBicg = 0
    for cfg in ("SellpTmaCfgILi4ELi3ELi16ELi1E", "SellpTmaCfgILi2ELi5ELi24ELi1E"):
        (k,) = _pick(sass, "sellp64_tma_kernel", cfg, "Lb0ELb0ELi0E")
        assert not ATOMIC.search(sass[k])
        assert "UBLKCP" in sass[k]
        assert "DMUL" in sass[k] and "DADD" in sass[k] and "DFMA" not in sass[k]  # separately rounded fold


def test_ell_and_csr_rowblock_spmv_have_no_atomics(sass):
    for k in _pick(sass, "ell_tma_kernel", "Lb0EE"):
        assert not ATOMIC.search(sass[k]), k
    for k in _pick(sass, "csr_rowblock_kernel"):
        assert not ATOMIC.search(sass[k]), k


def test_coo_kernel_uses_atomics(sass):
    ks = _pick(sass, "seg8_kernelILb0E")
    assert any(ATOMIC.search(sass[k]) for k in ks)


def test_radix_sort_downsweep_streams_with_tma(sass):
    """The ingestion sort's downsweep stages its sub-tiles with cp.async.bulk
    (UBLKCP) and ranks with ballots (VOTE), not match.any (MATCH)."""
    (k,) = _pick(sass, "rs_downsweep")
    assert "UBLKCP" in sass[k]
    assert "VOTE" in sass[k] and "MATCH" not in sass[k]


def test_csr_short_kernel_is_a_plain_fold(sass):
    """config-1 CSR kernel: separately rounded fold, no atomics."""
    (k,) = _pick(sass, "csr_short_kernel")
    assert not ATOMIC.search(sass[k])
    assert "DMUL" in sass[k] and "DADD" in sass[k] and "DFMA" not in sass[k]
