"""CPU oracle for the voxpar hot path -- TEST INFRASTRUCTURE ONLY.

A restatement of the reference's serial algorithm (reference
pkg/src/voxpar/layers/reference.py, model/serial.py, model/optim.py,
prng.py, kernels/_hot.pyx) in numpy + plain C (conv_oracle.c).  It is the
checker the CUDA path is compared against; only tests/, the smoke() entry
and bench.py's cpu_baseline leg may import it.  The product package
(paper_2007_12856_b200) never imports anything from here.

Pinning: tests/test_oracle.py checks this oracle against golden vectors in
tests/golden/ produced by running the reference itself
(tests/golden/make_golden.py) and, where built, bit-for-bit against the
reference's own compiled Cython kernels (oracle/_ref, oracle/build_oracle.py).
"""
