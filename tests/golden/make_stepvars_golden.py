"""Golden vectors for the analysis outputs of `fixed_point_step` (the slack `s` and the
spherical variables `vars` of its INPUT iterate, pkg/src/swarmplan/solver.py:246-256 ->
_analyze :158-169, extract_spherical constraints.py:195-213), by running the REFERENCE.

    python tests/golden/make_stepvars_golden.py     # writes tests/golden/stepvars_*.npz

The inputs are the S1-style random states of make_golden.py's step_* cases
(trainer/tests/test_acceptance.py:35-87) plus an 8-robot naive-prior batch.
"""

from __future__ import annotations

import os
import sys

sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

import numpy as np  # noqa: E402
from swarmplan.basis import BasisConfig, build_basis  # noqa: E402
from swarmplan.constraints import assemble  # noqa: E402
from swarmplan.pipeline import sample_naive_prior  # noqa: E402
from swarmplan.scenario import ScenarioFamily, generate  # noqa: E402
from swarmplan.solver import (ObjectiveMode, SolverConfig, SolverState, fixed_point_step,  # noqa: E402
                              stack_xi)

OUT = os.path.dirname(os.path.abspath(__file__))


def save(name, sys_, st, tgt, nxt):
    d = sys_.dims
    v = nxt.vars
    np.savez_compressed(
        os.path.join(OUT, f"stepvars_{name}.npz"),
        dims=np.array([d.n, d.n_d, d.n_basis, d.num_steps, d.n_obs, d.a_rows, d.g_rows]),
        W=sys_.basis.W, Wd=sys_.basis.Wd, Wdd=sys_.basis.Wdd, grid=sys_.basis.grid,
        duration=sys_.basis.config.duration,
        A=sys_.A, b=sys_.b, h=sys_.h, pair_axes=sys_.pair_axes, obs_axes=sys_.obs_axes,
        obs_pos=sys_.obs_pos, d_max=sys_.d_max, xi0=st.xi, lam0=st.lam, target=tgt,
        out_xi=nxt.xi, out_lam=nxt.lam, out_s=nxt.s,
        alpha=v.alpha, beta=v.beta, d=v.d, alpha_o=v.alpha_o, beta_o=v.beta_o, d_o=v.d_o)
    print(f"stepvars_{name}: n={d.n} m={d.n_obs} nd={d.n_d} B={st.xi.shape[-1]}")


def main():
    B50 = build_basis(BasisConfig())
    for label, scn in (("2d_obstacles", generate(ScenarioFamily("random_box", n_obstacles=2),
                                                 n=3, n_d=2, seed=2)),
                       ("3d", generate(ScenarioFamily("random_box", n_obstacles=1), n=3, n_d=3, seed=3))):
        sys_ = assemble(scn, B50)
        d = sys_.dims
        rng = np.random.default_rng(5)
        xi = 0.5 * rng.standard_normal((d.n_d, d.nvar_ax, 4))
        lam = 0.5 * rng.standard_normal((d.n_d, d.nvar_ax, 4))
        tgt = 0.3 * rng.standard_normal(xi.shape)
        st = SolverState(xi=xi, lam=lam)
        save(label, sys_, st, tgt, fixed_point_step(st, sys_, ObjectiveMode.projection(tgt),
                                                    SolverConfig()))
    fam = ScenarioFamily("random_box", robot_radius=0.1, box=(-1.5, 1.5), n_obstacles=3)
    scn = generate(fam, 8, 2, seed=11, horizon=B50.config)
    sys_ = assemble(scn, B50)
    xi = stack_xi(sample_naive_prior(scn, B50, 3, seed=11).candidates)
    st = SolverState(xi=xi, lam=np.zeros_like(xi))
    save("obs8", sys_, st, xi, fixed_point_step(st, sys_, ObjectiveMode.projection(xi), SolverConfig()))


if __name__ == "__main__":
    main()
