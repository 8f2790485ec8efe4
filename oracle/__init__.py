"""CPU oracle for the ZipPIR server hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package, and only as the checker (or, for the
bench, as the timed CPU baseline). The product package
(paper_2603_09190_b200) never imports it and has no CPU fallback.

Modules:
  ref.py       -- exact numpy / Python-int restatement of the reference's
                  server path (protocol.py, paillier.py, prg.py), each
                  function citing the reference file:line it follows.
  client.py    -- client-side restatement (keygen, query, decrypt, extract)
                  used only to manufacture test inputs.
  ref_port.py  -- restatement of the reference's own CPU *algorithm*
                  (centered float64 BLAS GEMV + 240-prime RNS engine) used as
                  the timed CPU baseline ("kind": "port").
  c/           -- plain-C restatement of the integer GEMV / hint product
                  (OpenMP), the fast checker at BASELINE sizes.

Parity pinning: tests/test_oracle_golden.py checks every function here
against tests/golden/*, which tests/golden/make_golden.py produced by running
the unmodified reference package (with a gmpy2 stand-in) in the build
container.
"""
