"""PCG golden cases (must mirror tests/golden/make_golden.py:case_pcg)."""
PCG_CASES = {
    "id_true": ("id", dict(rtol=1e-8)),
    "jac_true": ("jac", dict(rtol=1e-8)),
    "jac_delta": ("jac", dict(rtol=1e-10, termination="delta")),
    "id_max3": ("id", dict(max_iters=3)),
    "id_p7": ("id", dict(rtol=1e-10, period=7)),
    "zero_rhs": ("id", dict()),
    "learn_true": ("learn", dict(rtol=1e-8)),
    "learn_p3": ("learn", dict(rtol=1e-9, period=3)),
    "learn_delta": ("learn", dict(rtol=1e-9, termination="delta")),
}
