import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O
from paper_2108_05665_b200 import _abi as A
from paper_2108_05665_b200.engine import Engine, EvalOptions
from tests.helpers import random_instance
eng = Engine(0)
for seed in (3, 6, 9, 12, 15, 0, 1, 11):
    p, _, _ = random_instance(seed)
    want = O.eval_problem(p)[0]
    res = []
    for chunk in (1, 2, 3, 4):
        got = eng.eval(p, A.MTCG_EVAL_AUTO, EvalOptions(precision="c128", row_chunk=chunk)).amplitudes
        res.append(bool(np.array_equal(got, want)))
    print(seed, "sliced", len(p.sliced), "requests", p.n_requests, res, flush=True)
