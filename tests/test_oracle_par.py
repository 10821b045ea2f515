"""The process-parallel oracle driver (oracle/par.py) changes no number: its
fhat, treecode and direct sums are bitwise those of the single-process oracle
(it only splits cluster ranges / target slices over workers)."""
import numpy as np

import kitc_inputs as KI
import oracle as O
from oracle.par import ParOracle


def test_par_oracle_bitwise_serial():
    X, W = KI.particles(6000, seed=21)
    T = O.Tree(X, 120)
    F = T.modified_weights(W, 5)
    tg = KI.sample_targets(6000, 333, seed=2)
    ref, rst = T.treecode(0, 0.01, 5, 0.7, W, fhat=F, targets=tg, stats=True)
    dref = O.direct(0, 0.01, X, W, targets=tg[:50])
    with ParOracle(X, W, 120, procs=3) as P:
        assert P.tree.nclusters == T.nclusters
        G = P.modified_weights(5)
        assert np.array_equal(G, F)
        got, gst = P.treecode(0, 0.01, 5, 0.7, G, tg, stats=True)
        assert np.array_equal(got, ref) and np.array_equal(gst, rst)
        assert np.array_equal(P.direct(0, 0.01, tg[:50]), dref)
