"""CPU oracle for xGR's xBeam decode-step selection (section 6).

TEST INFRASTRUCTURE ONLY. Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` / `--impl reference` legs may import, call or execute anything in this package.
The product path (`paper_2512_11529_b200/`) never imports it, and the oracle imports nothing from
the product path: the two share no code, only the seeded generators in `synth/`.

Modules
  xbeam_oracle  plain definition in fp64 (numpy): trie, legal-only log-softmax, score add,
                full-sort global top-BW with the lower-flat-index tie-break, finalize.
  paper_heap    the paper's own selection procedure (section 6.2): a global
                min-heap of size BW with per-beam early termination; a second, independent
                selection oracle.
  brute         pure-Python enumeration for tiny tries (legal set by enumerating all V^ND tuples,
                path scores of every item by math.exp / math.log loops).
  kv_reorder    the unshared KV-cache reorder after a step (NEXT f2).
  attention     staged shared/unshared decode attention and its OnlineSoftmax merge (PAPER.md
                L339; NEXT f4's second workload), fp64.

Parity status of every function: pinned (see tests/test_oracle_pins.py and DESIGN.md section
"Oracle pins"). The pruned fraction and throughput numbers are parity-unpinned: the paper prints
none for this path.
"""
