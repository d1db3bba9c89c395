"""CPU oracle for the MagicDec self-speculative decode hot path (arXiv 2408.11049).

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import anything here.
The product path (`paper_2408_11049_b200`, the CUDA library) never imports,
links or executes this package, and this package never imports the product
path: the two share no code.  The one shared module is `synth/` (seeded input
generators, which hold none of the method's arithmetic).

Every function is the plain definition written out in fp64 (numpy), citing the
PAPER.md passage it follows (`P:<line>`, /root/reference/PAPER.md), plus the
reading of SURVEY.md §8(c) where the paper is silent (ledger in DESIGN.md §3).
MagicDec is exact ("lossless" SD): it changes what is drafted, not
the result, so attention is dense softmax over the defined index set and
acceptance is the speculative-sampling rule of Leviathan et al. that P:204 cites.

Modules
  attention  O1-O3, O6  : verify (full KV, causal over the gamma+1 rows, GQA),
                          draft (StreamingLLM sink + window), kv_append, split merge
  accept     O4         : speculative acceptance, SAMPLE and GREEDY modes
  philox     O5         : Philox4x32-10 counter-based uniforms
  theory     Eq.1       : expected generation length and accepted-count PMF
  enumerate  O4 pins    : exact rational output distribution on tiny vocabularies
  snapkv     f2         : SnapKV selection (votes, pooling, top-k) and index-list draft attention
  tree       f3         : tree-masked verify, tree acceptance, KV compaction
  pqcache    f4         : PQ encode, fixed-point lookup-table scores, exact top-k selection

Parity pins: every function is pinned in tests/test_oracle_*.py; see DESIGN.md
§4 for the list.  No function here is "parity unpinned".
"""
