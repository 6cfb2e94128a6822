import sys, os, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2202_07798_b200 import brbpnn
from oracle import bbml_oracle as O
for d, h, n, ep in ((2, 12, 40, 6), (2, 10, 40, 6), (1, 33, 40, 4)):
    X = np.random.default_rng(n + d).uniform(0, 1, size=(n, d))
    y = np.sin(3 * X.sum(axis=1))
    fit = O.br_fit(X, y, d, h, seed=3, max_epochs=ep)
    model, hist = brbpnn.train(X, y, hidden=h, seed=3, config=brbpnn.LmConfig(max_epochs=ep))
    print("case", d, h, n, "P=", h*(d+2)+1)
    for r_o, r_d in zip(fit.records, hist):
        print(" oracle", ["%.10g" % v for v in r_o[1:9]])
        print(" device", ["%.10g" % v for v in (r_d.f_before, r_d.f_after, r_d.e_d, r_d.e_w, r_d.alpha, r_d.beta, r_d.gamma, r_d.mu)])
