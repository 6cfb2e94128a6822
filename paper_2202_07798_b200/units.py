"""Device implementations of the reference's unit-level functions (the ones
its own tests call directly): pnn.loss_and_grads / adam_step, brbpnn.tansig,
jacobian, objective, solve_damped, evidence_update.  Thin wrappers over the
C-ABI unit kernels; host code only moves arrays and makes the (scalar)
control decisions the reference makes in Python.
"""

from __future__ import annotations

import numpy as np

from . import engine
from ._lib import PRED_TASK, check, lib, ptr


def _dev(torch, a, dtype=None):
    a = np.ascontiguousarray(a, dtype=np.float64 if dtype is None else dtype)
    return torch.from_numpy(a).to("cuda")


def _stream(torch):
    return torch.cuda.current_stream().cuda_stream


def _task(n, d, h, eps=1e-8):
    t = np.zeros(1, dtype=PRED_TASK)
    t["n"], t["d"], t["h"], t["eps"] = n, d, h, eps
    t["norm_offset"] = -1
    return t


def pnn_loss_grad(w, X, y, d, h, eps, nll_eps):
    torch = engine.torch_cuda()
    t = _task(len(y), d, h, eps)
    Xd, yd, wd = _dev(torch, X), _dev(torch, y), _dev(torch, w)
    loss = torch.empty(1, dtype=torch.float64, device="cuda")
    g = torch.empty(len(w), dtype=torch.float64, device="cuda")
    check(lib().bbml_pnn_loss_grad(ptr(t), 1, ptr(Xd), ptr(yd), X.shape[1], ptr(wd),
                                   float(nll_eps), ptr(loss), ptr(g), _stream(torch)),
          "bbml_pnn_loss_grad")
    return float(loss.cpu()[0]), g.cpu().numpy()


def adam_step(state, params: dict, grads: dict):
    """Mutates ``params`` (numpy arrays, in place) and ``state``; returns the
    name of the first block with a non-finite gradient or None."""
    torch = engine.torch_cuda()
    names = list(params.keys())
    sizes = [np.asarray(params[k]).size for k in names]
    begin = engine.offsets(np.array(sizes))
    flat = lambda src: np.concatenate([np.ravel(np.asarray(src[k], dtype=np.float64))
                                       for k in names]) if names else np.zeros(0)
    p, g, m, v = (_dev(torch, flat(x)) for x in (params, grads, state.m, state.v))
    state.step += 1
    t = state.step
    bc1 = 1.0 - state.beta1 ** t
    bc2 = 1.0 - state.beta2 ** t
    bb = _dev(torch, begin, np.int64)
    bad = torch.empty(1, dtype=torch.int32, device="cuda")
    check(lib().bbml_adam_step(ptr(p), ptr(g), ptr(m), ptr(v), int(sum(sizes)), ptr(bb),
                               len(names), bc1, bc2, state.learning_rate, state.beta1, state.beta2,
                               state.eps, ptr(bad), _stream(torch)), "bbml_adam_step")
    ph, mh, vh = p.cpu().numpy(), m.cpu().numpy(), v.cpu().numpy()
    bad_i = int(bad.cpu()[0])
    for k, o, s in zip(names, begin, sizes):
        shape = np.shape(params[k])
        params[k][...] = ph[o:o + s].reshape(shape)
        state.m[k] = mh[o:o + s].reshape(shape).copy()
        state.v[k] = vh[o:o + s].reshape(shape).copy()
    return None if bad_i < 0 else names[bad_i]


def tansig(x):
    torch = engine.torch_cuda()
    a = np.asarray(x, dtype=np.float64)
    xd = _dev(torch, a.ravel())
    yd = torch.empty_like(xd)
    check(lib().bbml_tansig(ptr(xd), ptr(yd), a.size, _stream(torch)), "bbml_tansig")
    return yd.cpu().numpy().reshape(a.shape)


def br_eval(w, X, y, d, h, want_jac: bool):
    """(residuals, E_D, E_W, J or None) at packed weights w (device)."""
    torch = engine.torch_cuda()
    n = len(X)
    P = h * (d + 2) + 1
    t = _task(n, d, h)
    Xd, yd, wd = _dev(torch, X), _dev(torch, y), _dev(torch, w)
    r = torch.empty(max(n, 1), dtype=torch.float64, device="cuda")
    en = torch.empty(2, dtype=torch.float64, device="cuda")
    J = torch.empty(max(n * P, 1), dtype=torch.float64, device="cuda") if want_jac else None
    joff = np.zeros(1, dtype=np.int64)
    check(lib().bbml_lm_jacobian(ptr(t), 1, ptr(Xd), ptr(yd), d, ptr(wd), ptr(joff) if want_jac else 0,
                                 ptr(J), ptr(r), ptr(en), _stream(torch)), "bbml_lm_jacobian")
    e = en.cpu().numpy()
    Jh = J.cpu().numpy()[:n * P].reshape(n, P) if want_jac else None
    return r.cpu().numpy()[:n], float(e[0]), float(e[1]), Jh


def gram(J, r):
    torch = engine.torch_cuda()
    n, P = J.shape
    Jd, rd = _dev(torch, J), _dev(torch, r)
    jtj = torch.empty(P * P, dtype=torch.float64, device="cuda")
    jtr = torch.empty(P, dtype=torch.float64, device="cuda")
    z = np.zeros(1, dtype=np.int64)
    Pa, na = np.array([P], np.int32), np.array([n], np.int32)  # keep alive across the call
    check(lib().bbml_lm_gram(ptr(Pa), ptr(na), 1,
                             ptr(z), ptr(z), ptr(z), ptr(z), ptr(Jd), ptr(rd), ptr(jtj), ptr(jtr),
                             _stream(torch)), "bbml_lm_gram")
    return jtj, jtr


def damped_solve(J, r, w, alpha, beta, mu):
    """(delta, singular?) for solve_damped (brbpnn.py:153-171)."""
    torch = engine.torch_cuda()
    J = np.atleast_2d(np.asarray(J, dtype=np.float64))
    P = J.shape[1]
    jtj, jtr = gram(J, np.asarray(r, dtype=np.float64))
    wd = _dev(torch, w)
    abm = _dev(torch, [alpha, beta, mu])
    delta = torch.empty(P, dtype=torch.float64, device="cuda")
    info = torch.empty(1, dtype=torch.int32, device="cuda")
    z = np.zeros(1, dtype=np.int64)
    Pa = np.array([P], np.int32)
    check(lib().bbml_lm_solve(ptr(Pa), 1, ptr(z), ptr(z), ptr(jtj), ptr(jtr),
                              ptr(wd), ptr(abm), ptr(delta), ptr(info), _stream(torch)),
          "bbml_lm_solve")
    return delta.cpu().numpy(), bool(int(info.cpu()[0]))


def evidence(e_d, e_w, jtj, alpha, beta, n_samples):
    """(alpha, beta, gamma, pinned, eigenvalues) for evidence_update."""
    torch = engine.torch_cuda()
    jtj = np.asarray(jtj, dtype=np.float64)
    P = jtj.shape[0]
    jd = _dev(torch, jtj.ravel())
    inp = _dev(torch, [e_d, e_w, alpha, beta, float(n_samples)])
    eig = torch.empty(P, dtype=torch.float64, device="cuda")
    out = torch.empty(5, dtype=torch.float64, device="cuda")
    z = np.zeros(1, dtype=np.int64)
    Pa = np.array([P], np.int32)
    check(lib().bbml_lm_evidence(ptr(Pa), 1, ptr(z), ptr(z), ptr(jd),
                                 ptr(inp), ptr(eig), ptr(out), _stream(torch)), "bbml_lm_evidence")
    o = out.cpu().numpy()
    return float(o[0]), float(o[1]), float(o[2]), bool(o[3]), np.sort(eig.cpu().numpy())
