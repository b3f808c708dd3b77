"""CPU oracle for the sparse fp64 hot path — TEST INFRASTRUCTURE ONLY.

This package restates, on the CPU, the algorithms of the reference package
`warpkit` (arXiv 2006.14290 workbench, `/root/reference/pkg/src/warpkit`)
that the B200 path replaces. It is the *checker*: only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s CPU-baseline / reference arm may
import it. The product package `paper_2006_14290_b200` never imports it and
has no CPU fallback.

Pinning: the restatements are checked against golden vectors produced by the
reference itself (`tests/golden/make_golden.py` imports warpkit in the build
container and writes `tests/golden/*.npz`). Items the reference does not
implement (ELL, Hybrid, BiCGSTAB, GMRES, load-balanced CSR) are "parity
unpinned" restatements from their textbook / Ginkgo definitions; see
DESIGN.md §Oracle.

Modules
  sparse_ref  formats, conversions, bitwise sequential SpMV fold
  krylov_ref  CG (exact restatement of kernels.py:283-331), BiCGSTAB, GMRES(m)
  corpus_ref  matrix generators (corpus.py restated + new 3-D / R-MAT families)
  native      ctypes binding of the C restatement (oracle/csrc/oracle.c), the
              all-cores CPU baseline
"""
