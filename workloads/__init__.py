"""Input producers for the tests and the bench — NOT the product.

`network.py` restates, bit for bit, the reference's caller-side producers
that SURVEY.md §2 marks out of scope (circuit parser and gate matrices,
circuit -> network diagram, build_assignments, plan parser, test
generators; proj/src/circuit.cpp, diagram.cpp, plan.cpp,
proj/tests/support/gen.cpp), plus the synthetic Sycamore-53 generator of
BASELINE configs 3-5. They exist so the GPU box — which has no reference
tree — can build the same inputs the reference would; they are pinned to the
reference in tests/test_network.py. The engine consumes their output through
the C ABI (include/mtcg.h) and never imports this package.
"""
