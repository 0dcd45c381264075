"""Mutation check of the oracle pins: every plausible mistake below, applied to a copy of
oracle/oracle.c, must make at least one `-m "not gpu"` oracle test fail.

    python tools/mutants.py            # all mutants, prints one line each, exit 1 if one survives

The mutants are the ones listed in the round-1 review plus the ones that
were already caught then.  Nothing here changes the oracle in the tree.
"""
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "oracle.c")
TESTS = ["tests/test_oracle_pins.py", "tests/test_oracle_sampling.py", "tests/test_oracle_entry.py",
         "tests/test_oracle_completion.py", "tests/test_oracle_mesh.py"]

MUTANTS = [
    ("g(j) = max instead of max - min (P:143)", "if (cnt[c]) g[c] = hi[c] - lo[c];", "if (cnt[c]) g[c] = hi[c];"),
    ("n_f with floor instead of ceil (P:104)", "double x = ceil(((double)in->nmax * lum) / lmax);",
     "double x = floor(((double)in->nmax * lum) / lmax);"),
    ("mixed pair drawn with n(I_f) instead of n(I_o) (R10)",
     "nb = orc_floyd(c->m, n_of(in, c->m, lum_node(in, o), lmax)",
     "nb = orc_floyd(c->m, n_of(in, c->m, lum_node(in, f), lmax)"),
    ("CDF inversion with >= (R29)", "if (cdf[mid] > x) hi = mid;", "if (cdf[mid] >= x) hi = mid;"),
    ("unobserved column weight = floor (R14)", "if (!cnt[c]) w[c] = wu;", "if (!cnt[c]) w[c] = 65536u;"),
    ("Eq. (1) with cost(a) added (P:112)", "double cf = eps + cost[b];", "double cf = eps + cost[b] + cost[a];"),
    ("weight floor 2^12 instead of 2^16 (R14)", "w[c] = wc > 65536u ? wc : 65536u;", "w[c] = wc > 4096u ? wc : 4096u;"),
    ("triangle: v + u bound dropped (R39)", "if (v < 0.0 || u + v > 1.0) return 0;", "if (v < 0.0 || v > 1.0) return 0;"),
    ("triangle: tmin ignored (R39)", "return t > tmin && t < tmax;\n}", "return t < tmax;\n}"),
    ("triangle: cross product sign (R39)", "c[1] = a[2] * b[0] - a[0] * b[2];", "c[1] = a[0] * b[2] - a[2] * b[0];"),
    ("triangle: e2 taken from v1 (R39)", "double e2[3] = {(double)tr[6] - v0[0]", "double e2[3] = {(double)tr[3] - v0[0]"),
]


def main():
    base = open(SRC).read()
    survivors = 0
    for name, old, new in MUTANTS:
        if base.count(old) != 1:
            print(f"SKIP  {name}: pattern not found once")
            survivors += 1
            continue
        with tempfile.TemporaryDirectory() as td:
            src = os.path.join(td, "oracle.c")
            open(src, "w").write(base.replace(old, new))
            so = os.path.join(td, "liboracle_mut.so")
            subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared",
                                   "-I", os.path.join(ROOT, "oracle"), "-o", so, src, "-lm"])
            env = dict(os.environ, ORACLE_LIB=so)
            r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "not gpu", "-p", "no:cacheprovider",
                                *TESTS], cwd=ROOT, env=env, capture_output=True, text=True)
            killed = r.returncode != 0
            last = [l for l in r.stdout.splitlines() if "FAILED" in l or "failed" in l]
            print(f"{'KILLED' if killed else 'SURVIVED'}  {name}   {last[0] if last else ''}")
            survivors += 0 if killed else 1
    print(f"{len(MUTANTS) - survivors} of {len(MUTANTS)} mutants killed")
    return 1 if survivors else 0


if __name__ == "__main__":
    sys.exit(main())
