#!/bin/bash
# Per-op decomposition of the complex64 tensor-core path's systematic scale
# error on cfg2 (tools/tc_bias.py): all tensor-core ops, each op alone
# (MTCG_TC_ONLY), and the CUDA-core path.
cd "$(dirname "$0")/.."
TC=0 python tools/tc_bias.py
python tools/tc_bias.py
MTCG_TC_KIND=tf32 python tools/tc_bias.py
for n in ${NODES:-279 337 329 319 311 291 299 285 227 275 102 191 213 134 262 116 135}; do
  MTCG_TC_ONLY=$n python tools/tc_bias.py
done
