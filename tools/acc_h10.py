"""Accuracy of the h = 10 BR fits (gramschmit series of suite16, random split)
against the oracle at a given epoch cap (development tool).
usage: python tools/acc_h10.py EPOCHS [--oracle]"""
import json, os, sys
from concurrent.futures import ProcessPoolExecutor
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

E = int(sys.argv[1])
from paper_2202_07798_b200 import synth
raw = [s for s in synth.suite16(seed=0) if s[0][0] == "gramschmit"]


def ora(item):
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    from oracle import bbml_oracle as O
    k, X, y = item
    r = O.train_one(k, X, y, "brbpnn", mode="random", base_seed=0, br_hidden=10, br_max_epochs=E)
    return None if r.error is not None else r.mse


if "--oracle" in sys.argv:
    with ProcessPoolExecutor(os.cpu_count()) as ex:
        m = list(ex.map(ora, raw))
    print(json.dumps({"who": "oracle", "mse": m}))
else:
    from paper_2202_07798_b200.experiment import ExperimentConfig, train_many
    from paper_2202_07798_b200.traces import BbSeries, SplitMode
    series = [BbSeries(k, X, y) for k, X, y in raw]
    cfg = ExperimentConfig(split_mode=SplitMode.RANDOM, seed=0, br_hidden=10, br_max_epochs=E,
                           models=("brbpnn",))
    res = train_many([(s, "brbpnn") for s in series], cfg).results
    print(json.dumps({"who": os.environ.get("BBML_LIB", "default"), "mse": [r.mse if r.error is None else None for r in res]}))
