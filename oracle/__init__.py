"""TEST INFRASTRUCTURE — parity checkers for the Brouwer–Zimmermann round.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference`` arm) may import this package. The
product (``paper_1911_08963_b200``) never does.

* ``oracle.ref``   — ctypes over ``oracle/_ref/libmdref*.so``: the UNMODIFIED
  reference C++ library (``/root/reference/proj/src``) plus our harness
  (``ref_harness.cpp``), built by ``oracle/Makefile``.
* ``oracle.port``  — ctypes over ``oracle/build/libmdoracle.so``: the plain-C
  restatement (``mdoracle.c``), pinned to the reference through
  ``tests/golden/``.
"""
