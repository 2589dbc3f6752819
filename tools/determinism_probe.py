"""Repeat one learner step from the same parameters on the same batch and report whether
the gradient is bit-identical across repeats (diagnostics)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2011_12895_b200 as tlg  # noqa: E402


def run(D, hidden, S, T, algo, reps=6):
    l = tlg.Learner("mlp", D, 6, hidden, algo=algo, optimizer="sgd", max_segments=S,
                    unroll_len=T)
    l.set_hyper(learning_rate=0.01, batch_size=S, unroll_len=T)
    p = tlg.synth.init_params_f32(l.n_params, 0.05, seed=3).astype(np.float64)
    b = tlg.synth.make_segments(S, T, D, 6, seed=4)
    gs = []
    for _ in range(reps):
        l.set_params(p)
        l.train_step(b)
        gs.append(l.get_grad())
    diffs = [float(np.max(np.abs(g - gs[0]))) for g in gs[1:]]
    print(f"D={D} hidden={hidden} S={S} T={T} {algo}: max |g - g0| over repeats {diffs} "
          f"(scale {np.max(np.abs(gs[0])):.3e})", flush=True)


if __name__ == "__main__":
    run(64, (512, 512), 256, 80, "vtrace")
    run(64, (256, 256), 64, 32, "ppo")
    run(64, (2048, 2048), 64, 64, "ppo_vtrace")
