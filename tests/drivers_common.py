"""The driver table shared by the CPU (bit-exact) and GPU (tolerance) tests;
mirrors the calls tests/golden/make_golden.py made with the reference."""

import numpy as np


def driver_runs(x30):
    from paper_1810_03358_b200.optimizers import (
        StopCriteria, cg, fgm, gradient_descent_fixed, heavy_ball, lbfgs, make_linesearch,
        nesterov_momentum, nesterov_strongly_convex, ofgm, steepest_descent)

    st40 = StopCriteria(max_iterations=40, gradient_norm_rtol=0.0)
    runs = {
        "sd_h": lambda o: steepest_descent(o, x30, make_linesearch("h"), st40),
        "sd_par": lambda o: steepest_descent(o, x30, make_linesearch("par"), st40),
        "gd": lambda o: gradient_descent_fixed(o, x30, 4000.0, st40),
        "hb": lambda o: heavy_ball(o, x30, 1.0 / 4000.0, 0.5, st40),
        "nag": lambda o: nesterov_momentum(o, x30, 4000.0, st40),
        "nagsc": lambda o: nesterov_strongly_convex(o, x30, 4000.0, 40.0, st40),
        "fgm": lambda o: fgm(o, x30, make_linesearch("par"), st40),
        "ofgm_L": lambda o: ofgm(o, x30, 40, L=4000.0, stop=st40),
        "ofgm_ls": lambda o: ofgm(o, x30, 40, linesearch=make_linesearch("h"), stop=st40),
        "lbfgs": lambda o: lbfgs(o, x30, m=4, linesearch=make_linesearch("h"), stop=st40),
    }
    for v in ("fr", "prp", "prp+", "hs", "cd", "ls", "dy"):
        runs["cg_" + v] = (lambda v: lambda o: cg(o, x30, v, make_linesearch("par"), st40))(v)
    return runs


def trace(res):
    f = np.array([r.f for r in res.trace.records])
    calls = np.array([[r.value_calls, r.grad_calls] for r in res.trace.records])
    return f, calls
