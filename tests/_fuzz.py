"""Seeded random configurations for the randomised GPU-vs-oracle parity checks (test helper; no
method arithmetic): tests/test_gpu_fuzz.py runs a committed subset, tools/fuzz_many.py sweeps more."""
import dataclasses

import numpy as np

import scenegen

TAU = {"cornell": 1.0e-4, "interior": 1.0e-3, "mesh": 1.0e-3}


def config_large(k):
    """larger slices and cuts (shared-memory and capacity edges), few iterations"""
    rng = np.random.default_rng(7_000_000 + k)
    kind = ["cornell", "interior", "mesh"][k % 3]
    nv = int(rng.integers(2000, 40000))
    cut = int(rng.integers(100, 1025))
    solver = int(rng.random() < 0.25)
    q = int(rng.choice([4, 8, 16, 32]))
    base = scenegen.PRESETS["t_mesh" if kind == "mesh" else "t_cornell" if kind == "cornell" else "t_interior"]
    return dataclasses.replace(
        base, name=f"fzL{k}", width=int(rng.integers(32, 129)), height=int(rng.integers(24, 97)), n_vpls=nv,
        cut_max=cut, slice_target=int(rng.integers(100, 1025)), rank_q=q, rate=float(rng.uniform(0.01, 0.3)),
        tau=TAU[kind] * float(rng.choice([0.0, 0.1, 1.0, 10.0])), solver=solver,
        max_iter=int(rng.integers(1, 6)), tol=0.0,
        row_importance=int(rng.random() < 0.3), cost_mode=int(rng.random() < 0.3),
        resolve_mode=int(rng.random() < 0.3),
        coarsen_target=int(rng.integers(1, cut + 1)) if rng.random() < 0.25 else 0,
        mesh_level=1 if kind == "mesh" else 0,
        seed=int(rng.integers(1, 2**62)), fixture_seed=int(rng.integers(1, 1000)))


def config_small(k):
    """small slices and cuts, every option, up to 40 iterations"""
    rng = np.random.default_rng(5_000_000 + k)
    kind = ["cornell", "interior", "mesh"][k % 3]
    nv = int(rng.integers(64, 20000))
    cut = int(rng.integers(2, min(nv, 400) + 1))
    solver = int(rng.random() < 0.25)
    q = int(rng.choice([4, 8, 16, 32]))
    base = scenegen.PRESETS["t_mesh" if kind == "mesh" else "t_cornell" if kind == "cornell" else "t_interior"]
    return dataclasses.replace(
        base, name=f"fz{k}", width=int(rng.integers(4, 97)), height=int(rng.integers(3, 81)), n_vpls=nv,
        cut_max=cut, slice_target=int(rng.integers(8, 301)), rank_q=q, rate=float(rng.uniform(0.01, 1.0)),
        tau=TAU[kind] * float(rng.choice([0.0, 0.1, 1.0, 10.0])), solver=solver,
        max_iter=int(rng.integers(1, 41)), tol=float(rng.choice([0.0, 0.0, 1e-2])),
        row_importance=int(rng.random() < 0.3), cost_mode=int(rng.random() < 0.3),
        resolve_mode=int(rng.random() < 0.3), p1_nmax=int(rng.choice([32, 32, 8, 16])),
        p1_nmin=int(rng.choice([4, 1, 2])),
        coarsen_target=int(rng.integers(1, cut + 1)) if rng.random() < 0.25 else 0,
        mesh_level=int(rng.choice([1, 2])) if kind == "mesh" else 0,
        seed=int(rng.integers(1, 2**62)), fixture_seed=int(rng.integers(1, 1000)))


def config_tiny(k):
    """degenerate sizes: 1-3 node cuts, 1-8 row slices, images of a few pixels"""
    rng = np.random.default_rng(9_000_000 + k)
    kind = ["cornell", "interior", "mesh"][k % 3]
    nv = int(rng.integers(1, 50))
    cut = int(rng.integers(1, min(nv, 3) + 1))
    solver = int(rng.random() < 0.3)
    base = scenegen.PRESETS["t_mesh" if kind == "mesh" else "t_cornell" if kind == "cornell" else "t_interior"]
    return dataclasses.replace(
        base, name=f"fzT{k}", width=int(rng.integers(1, 9)), height=int(rng.integers(1, 9)), n_vpls=nv,
        cut_max=cut, slice_target=int(rng.integers(1, 9)), rank_q=int(rng.choice([4, 8, 16, 32])),
        rate=float(rng.uniform(0.01, 1.0)), tau=TAU[kind] * float(rng.choice([0.0, 1.0, 100.0])), solver=solver,
        max_iter=int(rng.integers(1, 20)), p1_nmax=int(rng.choice([1, 2, 32])), p1_nmin=1,
        coarsen_target=1 if rng.random() < 0.3 else 0, mesh_level=1 if kind == "mesh" else 0,
        seed=int(rng.integers(1, 2**62)), fixture_seed=int(rng.integers(1, 1000)))


# configurations that exposed bugs (kept as regression cases): an odd cut size misaligned the u64
# CDF in k_pass2's shared memory; a mixed pair whose original child is brighter than every base
# pair needs a Floyd draw of more than 32 rows
REGRESSIONS = [
    scenegen.Config(name="reg_odd_cut", scene="mesh", width=34, height=46, n_vpls=1415, cut_max=75,
                    slice_target=192, rank_q=16, rate=0.198744968096291, tau=0.001, max_iter=31,
                    seed=304382001959307735, fixture_seed=592, resolve_mode=1, mesh_level=1),
    scenegen.Config(name="reg_floyd_gt32", scene="cornell", width=48, height=54, n_vpls=4770, cut_max=41,
                    slice_target=48, rank_q=16, rate=0.5970045329727259, tau=3e-05, solver=1, max_iter=35,
                    seed=4321912237893536051, fixture_seed=240, cost_mode=1),
]
