"""Race stress of the kernel's concurrency protocols by timing perturbation (compute-sanitizer
is closed on this GPU pool):

    python tools/race_stress.py [seeds] [--out DIR]

Every case runs once with the product library (libsfb.so) and once per jitter seed with
libsfb_checks.so (-DSFB_CHECKS: device asserts on the protocol invariants, and at the
exchange / handoff / task points a warp sleeps a seeded pseudo-random 0..~4 us). Any race in
the DSMEM exchange's parity-reused buffers, the split schedule's handoff or the task loop's
barriers would change a result under some interleaving; all results must be bitwise equal.
Cases: C3-shaped members over 2-, 4- and 8-CTA clusters (early exit on, so members leave
at different iterations), the split schedule (300 members > 296 resident CTAs, fixed and
early-exit), and the n = 40 16-warp build. Exit code 1 on any mismatch."""
import json
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASES = ["cluster2", "cluster4", "cluster8", "split_fixed", "split_exit", "wide40"]


def child(case, out):
    sys.path.insert(0, ROOT)
    import numpy as np
    from paper_2510_09204_b200 import solver
    from paper_2510_09204_b200.problem import (BasisConfig, ScenarioFamily, assemble, build_basis,
                                               generate, sample_naive_prior, stack_xi)

    def batch(n, m, inst, samples, seed=3000):
        basis = build_basis(BasisConfig(11, 100, 5.0))
        fam = ScenarioFamily("random_box", robot_radius=0.1, box=(-2.0, 2.0), n_obstacles=m)
        systems, xs = [], []
        for i in range(min(inst, 8)):
            scn = generate(fam, n, 2, seed=seed + i, horizon=basis.config)
            systems.append(assemble(scn, basis))
            xs.append(solver.to_member_major(stack_xi(sample_naive_prior(scn, basis, samples, seed=seed + i)), n, 11))
        reps = [i % len(systems) for i in range(inst)]
        xi = np.concatenate([xs[r] for r in reps])
        return [systems[r] for r in reps], xi, np.repeat(np.arange(inst), samples).astype(np.int32)

    if case.startswith("cluster"):
        s, x, mi = batch(32, 20, 2, 4)
        kw = dict(cfg=solver.SolverConfig(max_iters=60, primal_tol=1.5), cluster=int(case[-1]))
    elif case == "split_fixed":
        s, x, mi = batch(32, 20, 75, 4)
        kw = dict(cfg=solver.SolverConfig(max_iters=30), fixed_iterations=True, cluster=1)
    elif case == "split_exit":
        s, x, mi = batch(32, 20, 75, 4)
        kw = dict(cfg=solver.SolverConfig(max_iters=30, primal_tol=1.9), cluster=1)
    else:
        s, x, mi = batch(40, 12, 2, 2)
        kw = dict(cfg=solver.SolverConfig(max_iters=20), fixed_iterations=True, cluster=1)
    r = solver.solve_instances(s, x, None, x, member_instance=mi, **kw)
    np.savez(out, xi=r.xi, lam=r.lam, its=r.iterations, primal=r.primal,
             trace=np.concatenate([t.reshape(-1) for t in r.trace]))


def main():
    if len(sys.argv) > 2 and sys.argv[1] == "--child":
        child(sys.argv[2], sys.argv[3])
        return 0
    seeds = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 4
    checks = os.path.join(ROOT, "paper_2510_09204_b200", "libsfb_checks.so")
    if not os.path.exists(checks):
        print("libsfb_checks.so missing: run paper_2510_09204_b200.build.build_checks()")
        return 2
    import numpy as np
    bad = 0
    report = {}
    with tempfile.TemporaryDirectory() as tmp:
        for case in CASES:
            runs = [("plain", None, None)] + [("checks", checks, str(k + 1)) for k in range(seeds)]
            outs, times = [], []
            for label, lib, seed in runs:
                env = dict(os.environ)
                env.pop("SFB_JITTER_SEED", None)
                if lib:
                    env["SFB_LIB"] = lib
                    env["SFB_JITTER_SEED"] = seed
                out = os.path.join(tmp, f"{case}_{label}_{seed}.npz")
                t0 = time.perf_counter()
                p = subprocess.run([sys.executable, os.path.abspath(__file__), "--child", case, out], env=env,
                                   capture_output=True, text=True, timeout=900)
                times.append(round(time.perf_counter() - t0, 2))
                if p.returncode != 0:
                    print(f"{case} {label} seed={seed}: FAILED rc={p.returncode}\n{p.stderr[-1500:]}")
                    bad += 1
                    outs.append(None)
                    continue
                outs.append(np.load(out))
            ref = outs[0]
            same = []
            for o in outs[1:]:
                same.append(o is not None and ref is not None and
                            all(np.array_equal(o[k], ref[k]) for k in ref.files))
            ok = all(same)
            bad += 0 if ok else 1
            report[case] = {"seeds": seeds, "bitwise_equal": same, "process_seconds": times}
            print(f"{case:12s} {'PASS' if ok else 'FAIL'} — {seeds} jitter seeds, bitwise equal: {same}; "
                  f"process s (plain, seeds...): {times}", flush=True)
    print(json.dumps(report))
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
