"""Golden vectors for the GNN training step, from the REFERENCE package.

Runs in the build container only (needs /root/reference):
  * grad: one matrix's SAI loss and its tape gradient w.r.t. every parameter
    (training.py:_matrix_loss_and_grad: forward, Hutchinson probe from rng, sai_loss_on_tape,
    Tape.backward) for a random-init model on heat2d 8x8;
  * train: train() for 3 epochs (batch 4, AdamW, lr decay) on 8 heat2d 8x8 instances:
    per-epoch mean losses and the final flat parameters.
Writes tests/golden/golden_train.npz.
"""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

from spaigraph.datasets import gen_poisson2d  # noqa: E402
from spaigraph.gnn import GnnConfig, init_model  # noqa: E402
from spaigraph.graphfeat import build_graph  # noqa: E402
from spaigraph.training import TrainConfig, TrainItem, _matrix_loss_and_grad, train  # noqa: E402


def main():
    here = os.path.dirname(os.path.abspath(__file__))
    items = []
    for s in range(8):
        A, meta = gen_poisson2d(8, 8, coeff_seed=s)
        items.append(TrainItem(A, build_graph(A, meta)))
    out = {}
    model = init_model(GnnConfig(d_node=3, seed=0))
    out["params0"] = model.params_flat()
    rng = np.random.default_rng(123)
    loss, grad = _matrix_loss_and_grad(model, items[0], rng, TrainConfig())
    out["grad_loss"] = np.float64(loss)
    out["grad"] = grad
    cfg = TrainConfig(epochs=3, batch_size=4, seed=0)
    model2 = init_model(GnnConfig(d_node=3, seed=0))
    log = train(model2, items, cfg)
    out["train_losses"] = log.losses()
    out["train_lrs"] = np.array([r[2] for r in log.rows])
    out["train_params"] = model2.params_flat()
    np.savez_compressed(os.path.join(here, "golden_train.npz"), **out)
    print("grad loss", loss, "|grad|", float(np.linalg.norm(grad)), "train losses", log.losses())


if __name__ == "__main__":
    main()
