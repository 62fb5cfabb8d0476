"""ORACLE -- TEST INFRASTRUCTURE ONLY.

A CPU restatement of the reference's configuration-search path, used as the
parity checker for the CUDA product path.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline / ``--impl
reference`` legs may import it.  The product package
(``paper_2304_09781_b200``) never imports anything from here.

What it restates (reference file:line):
  * fleet feasibility                      mig.py:144-181 (C sum-set DP, feas.c)
  * FleetConfig decode                     mig.py:237-299
  * build_graph / ged / neighbours
  * table-surrogate evaluator, Eqs 1-3, 6  SPEC.md:411-449 (+ DESIGN.md surrogate)
  * accept rule / cooling / anneal
  * ORACLE exhaustive search, BLOVER draws SPEC.md:526-548, 553
  * derive_seed                            core.py:107-118

Pinning: feasibility and FleetConfig/partition semantics are pinned against
the reference's own code (exhaustive for n <= 6, tests/test_conformance.py and
tests/golden/*); the scalar Eq. 1/2/3/6/7 values against the SPEC's known-answer
examples.  The aggregate surrogate A(x), E(x), L(x) is this project's
definition (the SPEC's evaluator is an unimplemented DES): for those values
parity is "oracle == device, bit-exact", not "== reference".
"""
