"""CPU oracle for the layer-editing hot path -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.

``oracle.kn``   ctypes front-end of ``kn_port.c`` (C restatement of the reference's
                ``_kernels_numpy.py`` + the frozen definitions of the north-star ops).
``oracle.brute`` independent per-texel brute-force checkers (pure numpy / Python loops,
                small cases only) in the spirit of SPEC.md:62, 70, 283.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  ``paper_2501_14807_b200`` never does.
"""
