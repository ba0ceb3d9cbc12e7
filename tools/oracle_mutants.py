"""Mutation check of the oracle's pins: copy oracle/ to a scratch directory, apply one plausible
misreading at a time, and run the pin tests that must catch it.  Each mutant must fail at
least one test; the unmutated oracle must pass them all.

    python tools/oracle_mutants.py
"""
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SEL = ("box_and_mass or mass_energy or scaling_equivalence or covariance_M or reversible "
       "or energy_error")
# (name, file, old, new): each a single-site change of the oracle's leapfrog / HMC arithmetic
MUTANTS = [
    ("drift multiplies by M instead of M^-1", "__init__.py",
     "x = x + step * minv * p", "x = x + step / minv * p"),
    ("p0 = z sqrt(Minv) instead of z / sqrt(Minv)", "__init__.py",
     "hmc_normals(seed, it, x.size).reshape(x.shape) / np.sqrt(minv)",
     "hmc_normals(seed, it, x.size).reshape(x.shape) * np.sqrt(minv)"),
    ("reflection keeps the momentum (not an involution)", "__init__.py",
     "p = np.where(below | above, -p, p)", "p = p"),
    ("kinetic energy 1/2 sum p^2 / Minv", "__init__.py",
     "kin = 0.5 * float(np.sum(p * p * minv))", "kin = 0.5 * float(np.sum(p * p / minv))"),
    ("first half kick with the full step", "__init__.py",
     "p = p + 0.5 * step * g\n        x = x + step", "p = p + step * g\n        x = x + step"),
]


def run(oracle_dir):
    code = (f"import sys; sys.path.insert(0, {oracle_dir!r}); import oracle; import pytest; "
            f"sys.exit(pytest.main(['-q', 'tests/test_oracle_pins.py', '-k', {SEL!r}, "
            f"'-p', 'no:cacheprovider']))")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True)
    tail = [ln for ln in r.stdout.splitlines() if "passed" in ln or "failed" in ln]
    return r.returncode, tail[-1] if tail else r.stdout[-300:]


def main():
    bad = 0
    with tempfile.TemporaryDirectory() as d:
        base = os.path.join(d, "base")
        shutil.copytree(os.path.join(ROOT, "oracle"), os.path.join(base, "oracle"))
        rc, tail = run(base)
        print(f"unmutated: rc={rc} {tail}")
        bad += rc != 0
        for k, (name, fn, old, new) in enumerate(MUTANTS):
            m = os.path.join(d, f"m{k}")
            shutil.copytree(os.path.join(ROOT, "oracle"), os.path.join(m, "oracle"))
            p = os.path.join(m, "oracle", fn)
            src = open(p).read()
            assert src.count(old) == 1, f"mutant site not unique: {name}"
            open(p, "w").write(src.replace(old, new))
            rc, tail = run(m)
            print(f"mutant '{name}': {'caught' if rc != 0 else 'NOT CAUGHT'} ({tail})")
            bad += rc == 0
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
