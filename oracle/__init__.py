"""TEST INFRASTRUCTURE ONLY — CPU restatement of the reference hot path.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu-baseline / `--impl reference`
leg may import this package, and only as the checker or the CPU baseline.  The product
package `paper_2510_27517_b200` never imports it (a test enforces that).

Parity pin: `tests/golden/make_golden.py` runs the real reference (`/root/reference/pkg/src`,
importable in the build container) and commits its outputs as fixtures; `tests/test_oracle.py`
checks this restatement against those fixtures bit-for-bit (integer/pattern work) or to the
stated tolerance (floating point).
"""
