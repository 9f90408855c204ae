"""CPU oracle for the scoring hot path — TEST INFRASTRUCTURE ONLY.

This package restates, in plain numpy / Python, what the reference
(`metricforge` 0.1.0, mounted read-only at /root/reference during
development) computes on the path this repo accelerates:

* ``oracle.tokenizer``   greedy longest-match segmentation, per-kind
  sequence assembly and truncation   (ref ``pkg/src/metricforge/vocab.py``)
* ``oracle.batching``    window sort / mini-batch plan / inverse permutation
  (ref ``pkg/src/metricforge/batching.py``)
* ``oracle.encoder``     the fp32 and fp16-storage transformer encoder, BOS
  pooling, per-kind features and the tanh regression head
  (ref ``pkg/src/metricforge/encoder.py``)
* ``oracle.fixtures``    seeded fixture / synthetic-workload generators
  (ref ``pkg/tests/fixturegen.py`` plus SURVEY.md §8(d))
* ``oracle.mfrg``        an independent byte-level ``.mfrg`` container reader
  and writer (ref ``pkg/src/metricforge/container.py``)

Pinning: the oracle is checked against the reference's own golden file
``pkg/tests/golden/eval_qe.txt`` (copied as ``tests/golden/eval_qe.txt``) and
against vectors produced by running the reference itself in the development
container (``tests/golden/make_golden.py`` → ``tests/golden/*.json``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this package, and only as the checker / reported CPU baseline.
The product path (``paper_2408_11853_b200``) never imports it.
"""
