"""cvsr ORACLE -- plain fp64 CPU reference of the sliced-reconciliation hot path.

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import it.
It imports nothing from the CUDA package ``paper_2108_08418_b200`` and shares
no code with it.

Parity-pin status per function:
  quantise, slice_bits, syndrome  -- pinned (definition, brute force, invariants)
  llr_slice, llr_biawgn           -- pinned (closed forms, Monte Carlo, normalisation)
  bp_decode, bp_trace             -- pinned (tree exactness vs brute-force marginals,
                                     Hamming ML statistics, SPC/repetition closed forms,
                                     sign symmetry, (3,6) threshold trend)
  layers, bp_decode_layered       -- pinned (colouring validity + greedy minimality by brute
                                     force, tree exactness, repetition-chain sum, one-layer
                                     = flooding, Hamming ML statistics)
  bp_trace_layered                -- pinned through bp_decode_layered (same code path, fixed k)
  reconcile (both schedules)      -- pinned (tests/test_oracle_reconcile_pins.py: two-slice
                                     conditioning vs the two-bin closed form through an exactly
                                     solvable check, forced failure skips later slices (A-13),
                                     noiseless D = 0, one slice = the decoder, schedules agree)
  verify.frame_hash               -- pinned (key = 1 word checksum, key = 2^32 shifted
                                     integer, zero string, bit-flip detection)
  pa.toeplitz_hash                -- pinned (numpy convolution window, unit / all-ones
                                     seeds, linearity, 2-universality statistics)
"""
from .oracle import (  # noqa: F401
    build, bp_decode, bp_decode_layered, bp_trace, bp_trace_layered, layers, llr_biawgn, llr_slice, quantise, reconcile, slice_bits,
    syndrome, num_threads,
)
