"""Regenerate the trained-weights fixture with the REFERENCE trainer (test infrastructure).

Runs in the build container only (needs /root/reference).  Reproduces the reference's
acceptance-gate protocol (pkg/tests/test_acceptance.py:49-53, 85-103): 50 heat2d 16x16
instances (gen_poisson2d(16,16,coeff_seed=s), s=0..49), make_split(ratio=(4,1), seed=0),
init_model(GnnConfig(d_node=3)), train(model, items, TrainConfig()) with the defaults
(training.py:150-171).  Writes the SPAIGNN\\x01 checkpoint (gnn.py:270-289) to
tests/golden/trained_heat16.spaignn and prints the final mean loss.

The checkpoint is an INPUT to the hot path (weights), not an output under test.
"""
import hashlib
import os
import sys
import time

sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

from spaigraph.datasets import gen_poisson2d, make_split  # noqa: E402
from spaigraph.gnn import GnnConfig, init_model, save_checkpoint  # noqa: E402
from spaigraph.graphfeat import build_graph  # noqa: E402
from spaigraph.training import TrainConfig, TrainItem, train  # noqa: E402


def main():
    here = os.path.dirname(os.path.abspath(__file__))
    problems = []
    for s in range(50):
        A, meta = gen_poisson2d(16, 16, coeff_seed=s)
        problems.append((A, build_graph(A, meta)))
    train_p, _ = make_split(problems, (4, 1), seed=0)
    model = init_model(GnnConfig(d_node=3))
    t0 = time.time()
    log = train(model, [TrainItem(A, g) for A, g in train_p], TrainConfig())
    path = os.path.join(here, "trained_heat16.spaignn")
    save_checkpoint(model, path)
    blob = open(path, "rb").read()
    print("final_loss", repr(float(log.losses()[-1])), "seconds", round(time.time() - t0, 1))
    print("sha256", hashlib.sha256(blob).hexdigest())


if __name__ == "__main__":
    main()
