"""CPU oracle for the Sylvie halo path — TEST INFRASTRUCTURE ONLY.

This package restates, in numpy/scipy float64, the reference's algorithm for
the per-layer halo path (`halobit`, /root/reference/pkg/src/halobit):

* ``oracle.rng``     — key derivation + Philox4x64-10 uniform stream
                       (reference ``rngstream.py:19-39``);
* ``oracle.codec``   — per-row stochastic-rounding quantizer, LSB-first packing,
                       dequantizer, wire block layout (``codec.py:55-207``);
* ``oracle.epoch``   — a sequential, single-process restatement of the
                       distributed epoch (``trainer.py:175-372``,
                       ``transport.py:126-205``): halo exchange, Sylvie-S/A,
                       staleness adaptor, SpMM, GEMMs, CE, Adam, byte meters.

Who may use it: ``tests/`` (as the parity checker), ``__graft_entry__.smoke()``
(as the checker of one small CUDA call) and ``bench.py`` (the ``cpu_baseline``
leg and ``--impl reference``).  The product package
``paper_2303_01277_b200`` never imports it; its device path fails loudly if
the CUDA extension is missing.

Pinning: the restatement is checked against golden vectors produced by the
real reference in the build container (``tests/golden/make_golden.py``), see
``tests/test_oracle.py``.
"""
