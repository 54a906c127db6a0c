"""TEST INFRASTRUCTURE ONLY -- the CPU oracle for the B200 CKKS engine.

A restatement of the reference algorithm for the hot path (the CKKS engine
of /root/reference/pkg/src/hebert: _kernels.py -> ring.py -> ckks/*), in numpy
with an optional C/OpenMP kernel table (oracle/csrc/hekernels.c).  Every
function cites the reference file:line it follows.

Pinning: tests/test_oracle_golden.py checks the oracle against golden vectors
produced by running the reference itself (tests/golden/make_golden.py):
kernel outputs, NTTs, keygen digests, seeded encryptions, key switches,
rescales, products and rotations at N=2^6..2^16.  Parity is therefore pinned,
not self-referential.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may import
this package, and only as the checker / CPU baseline.  The product
(paper_2210_02574_b200) never imports it.
"""
