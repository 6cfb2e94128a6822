mkdir -p gpurun_out
nproc
(timeout 900 python tools/acc_h10.py 1000 --oracle > gpurun_out/acc_oracle.json 2>gpurun_out/acc_oracle.err) &
for l in ab/libbbml_base.so ab/libbbml_tri.so; do BBML_LIB=$l timeout 300 python tools/acc_h10.py 1000 > gpurun_out/acc_$(basename $l .so).json 2>&1; done
wait
python - <<'PY'
import json, numpy as np
o = np.array(json.load(open("gpurun_out/acc_oracle.json"))["mse"], dtype=float)
for n in ("libbbml_base", "libbbml_tri"):
    d = np.array(json.load(open(f"gpurun_out/acc_{n}.json"))["mse"], dtype=float)
    rel = np.abs(d - o) / np.maximum(np.abs(o), 1e-300)
    print(n, "acc dev %.3f oracle %.3f" % (100 * (1 - d.mean()), 100 * (1 - o.mean())),
          "rel mse diff median %.2e p90 %.2e max %.2e" % (np.median(rel), np.quantile(rel, 0.9), rel.max()),
          "|dmse| max %.2e" % np.abs(d - o).max())
PY
