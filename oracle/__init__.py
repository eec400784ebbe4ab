"""CPU oracle for the striped-attention hot path -- TEST INFRASTRUCTURE ONLY.

Nothing in ``paper_2311_09431_b200`` imports this package.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` leg may call it, and only as the checker or as the timed
CPU baseline -- never as the thing measured or shipped.

``ringref`` restates, in numpy, the reference ``ringsim`` package
(``/root/reference/pkg/src/ringsim``): token layouts (layout.py), block masks and
tile classification (attention.py), the streaming-softmax accumulator and the
N-round ring schedule (simulator.py).  Every function cites the reference
file:line it follows.

Pinning: the forward restatement (O, and LSE = m + ln l read from the
reference accumulator) is checked against golden vectors produced by running
the reference itself (``tests/golden/make_golden.py`` imports ringsim from
/root/reference in the build container and commits ``tests/golden/*.npz``).

Backward, multi-head / GQA and bf16 I/O have NO reference counterpart
(SPEC.md:14): ``ringref.dense_backward`` is the builder's fp64
restatement of the standard softmax-attention gradients, pinned by torch fp64
autograd of the reference's forward formula and by central finite differences
(tests/test_oracle_backward.py).  It is labelled "not reference" wherever used.
"""
