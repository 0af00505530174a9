"""CPU oracle -- TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference's hot path (jump_mppi, pure
Python/numpy; /root/reference/pkg/src/jump_mppi) used as the checker for the
GPU kernels.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline leg may import it; the product package never does.

Pinning: tests/test_oracle_golden.py checks this restatement against golden
vectors produced by running the reference itself in the build container
(oracle/gen_golden.py -> tests/golden/*.npz), and the Philox emulation against
the Random123 known-answer vectors.  Third-party arithmetic: numpy (>=1.24,
2.3.5 in this image) provides the reference's RNG (Philox4x64 + ziggurat
normals) and libm trig; `sample_noise_batch_ref` calls the same numpy
generator methods in the same order as noise.py:129-161, so it reproduces the
reference's noise bit for bit on the same numpy.
"""
