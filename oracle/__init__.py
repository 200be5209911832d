"""TEST INFRASTRUCTURE ONLY -- CPU oracle for the sketched Hessenberg / sLSLU loop.

Nothing in the product package (``paper_2502_02721_b200``) imports, links or
executes anything under this directory.  Only ``tests/``,
``__graft_entry__.smoke()`` and the ``cpu_baseline`` / ``--impl reference``
legs of ``bench.py`` may use it, and there only as the checker or the timed CPU
baseline -- never as the measured or shipped path.

Contents
--------
hessketch_oracle.py
    numpy restatement of the reference's per-iteration loop
    (``hessenberg.py`` init/step, ``solvers.py:_hessenberg_solve``,
    ``linops.py`` QR kernels, ``sketch.py`` PCG64 sketch), parametrised by the
    working precision (float64 = the reference; float32 = the "oracle32"
    restatement the fp32 device path is checked against).
tomo_oracle.py
    numpy restatement of the reference's parallel-beam ray tracer
    (``problems.py:_trace_ray`` / ``tomography_matrix``) generalised to a
    detector count different from the grid size, plus the operators the device
    kernels must reproduce bit for bit (sequential CSR row sums, tap-ordered
    PSF stencil, sequential dense rows).
coracle.c
    C restatement of the same loop (OpenMP over rows) used as the timed CPU
    baseline at sizes the numpy port cannot reach in seconds.

Pinning: ``tests/golden/make_golden.py`` runs the unmodified reference (only in
the build container, where ``/root/reference`` exists) and stores its outputs
as small ``.npz`` fixtures; ``tests/test_oracle_golden.py`` checks this oracle
against every fixture.
"""
