import sys, os, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2202_07798_b200 import brbpnn
from paper_2202_07798_b200.traces import BbSeries, SplitSpec, SplitMode, split, fit_normalizer
from paper_2202_07798_b200.experiment import series_seed
from oracle import bbml_oracle as O
g = np.load("tests/golden/train_one.npz")
for i in range(int(g["n_runs"])):
    p = f"r{i}_"; app, k, b, kind, mode = (str(v) for v in g[p + "key"])
    if (app, k, b, kind) != ("app20", "3", "3", "brbpnn"): continue
    seed, pe, be = (int(v) for v in g[p + "cfg"])
    s = BbSeries((app, int(k), int(b)), g[p + "X"], g[p + "y"])
    tr, te = split(s, SplitSpec({"high-low": SplitMode.HIGH_LOW, "random": SplitMode.RANDOM, "mixed-high-low": SplitMode.MIXED_HIGH_LOW}[mode], 0.7, seed))
    nm = fit_normalizer(tr); X = nm.transform_features(tr.X); y = nm.transform_targets(tr.y)
    sd = series_seed(seed, s.key, kind)
    print(mode, "n", len(y), "y uniq", np.unique(y), "seed", sd)
    fit = O.br_fit(X, y, 2, 1, seed=sd, max_epochs=be)
    model, hist = brbpnn.train(X, y, hidden=1, seed=sd, config=brbpnn.LmConfig(max_epochs=be))
    print("epochs oracle", len(fit.records), "device", len(hist))
    for e in range(min(len(hist), len(fit.records))):
        ro = fit.records[e]; rd = hist[e]
        if e < 6 or e > len(hist) - 4:
            print(e, "o", ["%.8g" % v for v in ro[1:9]], "\n  d", ["%.8g" % v for v in (rd.f_before, rd.f_after, rd.e_d, rd.e_w, rd.alpha, rd.beta, rd.gamma, rd.mu)])
    print("w oracle", fit.w, "\nw device", brbpnn.pack(model))
