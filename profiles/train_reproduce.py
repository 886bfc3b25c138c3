"""Reproduce the reference's trained fixture end to end with the GPU training step.

    python profiles/train_reproduce.py [--epochs 500]

Protocol of tests/golden/make_trained_fixture.py (the reference acceptance gate,
pkg/tests/test_acceptance.py:49-53, 85-103): 50 heat2d 16x16 systems, make_split((4, 1), seed 0),
init_model(GnnConfig(d_node=3)), train() with the TrainConfig defaults (500 epochs, batch 4).
The reference run ends at mean loss 27.94158728739968; prints one JSON line
with our final loss, its relative difference, the wall time and the steps/s.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

REFERENCE_FINAL_LOSS = 27.94158728739968


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--epochs", type=int, default=500)
    p.add_argument("--batched", action="store_true", help="one union graph per minibatch")
    a = p.parse_args()
    import paper_2510_27517_b200 as P
    from paper_2510_27517_b200.datasets import make_split
    problems = []
    for s in range(50):
        A, meta = P.gen_poisson2d(16, 16, coeff_seed=s)
        problems.append((A, P.build_graph(A, meta)))
    train_p, _ = make_split(problems, (4, 1), seed=0)
    model = P.init_model(P.GnnConfig(d_node=3))
    cfg = P.TrainConfig(epochs=a.epochs)
    t0 = time.perf_counter()
    log = P.train(model, [P.TrainItem(A, g) for A, g in train_p], cfg, batched=a.batched)
    wall = time.perf_counter() - t0
    final = float(log.losses()[-1])
    steps = a.epochs * len(train_p)
    out = {"what": "GPU training step, reference acceptance protocol", "batched": a.batched, "epochs": a.epochs,
           "matrices_per_epoch": len(train_p), "final_mean_loss": final, "wall_s": wall,
           "matrix_steps_per_s": steps / wall}
    if a.epochs == 500:
        out["reference_final_loss"] = REFERENCE_FINAL_LOSS
        out["rel_diff"] = abs(final - REFERENCE_FINAL_LOSS) / REFERENCE_FINAL_LOSS
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
