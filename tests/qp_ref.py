"""Reference QP for the projection: the problem the reference's acceptance test hands to
cvxpy (pkg/tests/test_acceptance.py:161-168), solved with scipy's SLSQP because cvxpy is
absent in this image.  Test infrastructure only."""

import numpy as np


def qp_reference(shot, a, b):
    """min ||s - shot||^2 s.t. |s| <= 1, |s[i+1] - s[i]| <= a, |s[i+2] - 2 s[i+1] + s[i]| <= b
    (the QP the reference hands to cvxpy, test_acceptance.py:161-168), by SLSQP."""
    from scipy.optimize import minimize

    n, d = shot.shape
    target = shot.ravel()

    def cons(x):
        s = x.reshape(n, d)
        d1 = s[1:] - s[:-1]
        d2 = s[2:] - 2 * s[1:-1] + s[:-2]
        return np.concatenate([a * a - np.sum(d1 * d1, 1), b * b - np.sum(d2 * d2, 1)])

    res = minimize(lambda x: np.sum((x - target) ** 2), np.clip(target, -1, 1),
                   jac=lambda x: 2 * (x - target), method="SLSQP",
                   bounds=[(-1.0, 1.0)] * (n * d), constraints=[{"type": "ineq", "fun": cons}],
                   options={"ftol": 1e-15, "maxiter": 1000})
    assert cons(res.x).min() >= -1e-9  # feasible (SLSQP may stop at its line-search floor)
    return res.x.reshape(n, d)
