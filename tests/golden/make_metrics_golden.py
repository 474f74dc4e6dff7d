"""Golden vectors of the post-solve metrics epilogue, made by running the REFERENCE's
`swarmplan.metrics.compute_metrics` (pkg/src/swarmplan/metrics.py:48-87).

Run in the dev container (the reference is mounted read-only at /root/reference):

    python tests/golden/make_metrics_golden.py      # writes tests/golden/metrics_*.npz

Each fixture holds a stack of trajectory sets coeffs (C, n, n_d, n_basis), the basis
config, the dense factor, the scenario's obstacles (center, velocity, radii as (n_obs, 3, 3),
zero padded to 3 axes) and the reference's five metrics per set (C, 5).
"""

from __future__ import annotations

import os
import sys

sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

import numpy as np  # noqa: E402
from swarmplan.basis import BasisConfig, build_basis, straight_line_coeffs  # noqa: E402
from swarmplan.metrics import compute_metrics  # noqa: E402
from swarmplan.pipeline import sample_naive_prior  # noqa: E402
from swarmplan.scenario import Obstacle, Scenario, ScenarioFamily, generate  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
FIELDS = ("smoothness", "arc_length", "min_pairwise_clearance", "avg_pairwise_distance",
          "min_obstacle_clearance")


def _obs_array(scn):
    arr = np.zeros((len(scn.obstacles), 3, 3))
    for o, ob in enumerate(scn.obstacles):
        arr[o, 0, : len(ob.center)] = ob.center
        arr[o, 1, : len(ob.velocity)] = ob.velocity
        arr[o, 2, : len(ob.radii)] = ob.radii
    return arr


def save(name, scn, cfg, coeffs, dense_factor=10):
    basis = build_basis(cfg)
    met = np.array([[getattr(compute_metrics(c, basis, scn, dense_factor), f) for f in FIELDS]
                    for c in coeffs])
    np.savez_compressed(os.path.join(OUT, f"metrics_{name}.npz"), coeffs=np.asarray(coeffs),
                        n_basis=cfg.n_basis, num_steps=cfg.num_steps, duration=cfg.duration,
                        dense_factor=dense_factor, n_d=scn.n_d, obstacles=_obs_array(scn),
                        metrics=met)
    print(name, met.shape)


def main():
    # C3-shaped: 32 robots, 20 static obstacles, noisy naive priors (pipeline.py:59-82)
    cfg = BasisConfig(11, 100, 5.0)
    scn = generate(ScenarioFamily("random_box", box=(-2.0, 2.0), n_obstacles=20), 32, 2,
                   seed=3000, horizon=cfg)
    cand = sample_naive_prior(scn, build_basis(cfg), 4, seed=3000).candidates
    save("c3_prior", scn, cfg, cand)
    # pipeline's ranking use: dense_factor = 1 (pipeline.py:133)
    save("c3_dense1", scn, cfg, cand[:2], dense_factor=1)
    # 3D, moving spheroids, few robots, default horizon
    cfg = BasisConfig(11, 50, 5.0)
    scn = generate(ScenarioFamily("random_box", box=(-1.5, 1.5), n_obstacles=2), 6, 3, seed=12,
                   horizon=cfg)
    obs = [Obstacle(center=o.center, radii=np.array([0.3, 0.3, 0.5]),
                    velocity=0.1 * np.arange(1, 4)[: scn.n_d] * (-1) ** k)
           for k, o in enumerate(scn.obstacles)]
    scn.obstacles = obs
    cand = sample_naive_prior(scn, build_basis(cfg), 3, seed=12).candidates
    save("d3_moving", scn, cfg, cand)
    # single robot, no obstacles (test_metrics.py:23-36): infinities, chord length
    scn1 = Scenario(n=1, n_d=2, radii=[0.1] * 3, starts=[[-1.0, 0.0]], goals=[[1.0, 0.0]],
                    obstacles=[], p_min=[-2, -2], p_max=[2, 2])
    line = straight_line_coeffs(scn1.starts, scn1.goals, 11)
    rng = np.random.default_rng(5)
    bent = line.copy()
    bent[:, :, 1:-1] += 0.3 * rng.standard_normal(bent[:, :, 1:-1].shape)
    save("single", scn1, BasisConfig(11, 50, 5.0), np.stack([line, bent]))
    # moderate n with odd sizes: 9 robots, 5 obstacles, n_basis 7, 37 steps, factor 3
    cfg = BasisConfig(7, 37, 3.0)
    scn = generate(ScenarioFamily("random_box", box=(-1.5, 1.5), n_obstacles=5), 9, 2, seed=21,
                   horizon=cfg)
    cand = sample_naive_prior(scn, build_basis(cfg), 2, seed=21).candidates
    save("odd", scn, cfg, cand, dense_factor=3)


if __name__ == "__main__":
    main()
