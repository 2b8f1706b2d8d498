"""CPU oracle for the array hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
arm may import this package, and only as the checker / the timed reference
port. The product path (``paper_2506_19656_b200``) never imports it.

* ``cubevid_oracle`` — numpy restatement of the reference's transform / cube /
  plan / planar-layout functions (each cites the reference file:line it
  follows); pinned against golden vectors produced by the reference itself
  (tests/golden/, script tests/golden/make_golden.py).
* ``metrics_oracle`` — float64 restatement of the absent metrics module
  (SPEC.md:400-477), pinned by SPEC's known answers and brute-force loops.
"""
