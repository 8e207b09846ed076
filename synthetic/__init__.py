"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This package holds NO arithmetic of the method (no snapping, no curl, no
spectral decomposition, no FFT operator, no eigensolver).  It only produces
problem *inputs* with the shapes and value distributions of the paper's
workloads (§6) as concretised in SURVEY.md §8(d):

* ``configs``  -- the five BASELINE.json configurations: raw primitive
  vectors, grid, Bloch vectors (Cartesian), number of eigenvalues.
* ``eps``      -- permittivity sampled at Yee edge midpoints, given a lattice
  geometry computed by the *caller* (oracle or library).
* ``vectors``  -- seeded random complex vectors for operator parity tests.
"""
