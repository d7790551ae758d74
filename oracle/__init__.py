"""CPU oracle for the B200 speculative-decoding step — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` legs may import this package, and only as the checker or as the timed CPU
baseline; the product path (``paper_2512_23858_b200``) never imports it and has no CPU
fallback.

Modules:
  tree_ref   restatement of the reference's tree / objective / acceptance / scheduling
             algorithms (pkg/src/specsim/{token_tree,egt,acceptance,latency,scheduler}.py),
             each function citing the file:line it follows.  Pinned against golden vectors
             generated from the reference itself (tests/golden/make_golden.py) and against the
             reference's own known-answer tests.
  llama_ref  torch-CPU fp32 Llama forward with KV cache and tree masks — the model arithmetic
             the reference does not have ("parity unpinned by the reference"
             for logits/attention/KV; pinned instead by the draft-independent identity
             "greedy speculative output == plain greedy AR decoding of the target").
  spec_ref   the whole speculative step on the CPU (draft passes, EGT growth, prune, verify,
             greedy walk, KV compaction) composed from the two modules above.
"""
