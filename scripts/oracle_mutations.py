"""Mutation check of the oracle's pins (tests -m "not gpu").

Each mutation is a plausible mistake in the oracle's MLS-MPM code (a wrong
constant, a dropped term, a wrong sign).  The script copies oracle/ to a
scratch directory, applies one mutation, rebuilds the copy and runs the oracle
pin tests against it; a mutation that every pin accepts is reported as
SURVIVED.  Usage: python scripts/oracle_mutations.py
"""
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = "oracle/sg_oracle.cpp"

MUTATIONS = [
    ("(none: the unmutated copy must pass)", "s4 = 4.0 * idx * idx", "s4 = 4.0 * idx * idx"),
    ("APIC scale 4/dx^2 -> 3/dx^2 (G2P)", "s4 = 4.0 * idx * idx", "s4 = 3.0 * idx * idx"),
    ("stress 4E -> 2E (P2G)", "double stress = -dt * 4.0 * E * pv", "double stress = -dt * 2.0 * E * pv"),
    ("affine term dropped (P2G)", "aff[r][c] = pm * A_(g, ar[2], 3 * r + c, i) +", "aff[r][c] = 0.0 * A_(g, ar[2], 3 * r + c, i) +"),
    ("J update sign (G2P)", "A_(g, ar[o0 + 3], 0, i) = J * (1.0 + dt * tr);", "A_(g, ar[o0 + 3], 0, i) = J * (1.0 - dt * tr);"),
    ("stress sign (P2G)", "double stress = -dt * 4.0", "double stress = dt * 4.0"),
    ("C transposed (G2P)", "nC[r][d] += s * gv;", "nC[d][r] += s * gv;"),
    ("middle B-spline weight (0.75 -> 0.7)", "k.w[1][a] = 0.75 -", "k.w[1][a] = 0.7 -"),
]

TESTS = ["tests/test_oracle_mpm.py", "tests/test_oracle_c4.py"]


def main():
    survived = []
    with tempfile.TemporaryDirectory() as tmp:
        for name, old, new in MUTATIONS:
            d = os.path.join(tmp, "m")
            if os.path.exists(d):
                shutil.rmtree(d)
            os.makedirs(d)
            shutil.copytree(os.path.join(ROOT, "oracle"), os.path.join(d, "oracle"),
                            ignore=shutil.ignore_patterns("*.so", "__pycache__"))
            p = os.path.join(d, SRC)
            s = open(p).read()
            assert s.count(old) >= 1, f"mutation anchor not found: {old}"
            open(p, "w").write(s.replace(old, new))
            env = dict(os.environ, PYTHONPATH=d + os.pathsep + ROOT)
            r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider"] +
                               [os.path.join(ROOT, t) for t in TESTS], cwd=d, env=env,
                               stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
            killed = r.returncode != 0
            first = next((ln.split(" ")[1] for ln in r.stdout.splitlines() if ln.startswith("FAILED")), "")
            if old == new:
                assert not killed, "the unmutated oracle copy fails its pins:\n" + r.stdout[-3000:]
                print(f"baseline  {name}")
                continue
            print(f"{'killed  ' if killed else 'SURVIVED'}  {name}  {first}")
            if not killed:
                survived.append(name)
    n = len(MUTATIONS) - 1
    print(f"{n - len(survived)}/{n} mutations killed")
    return 1 if survived else 0


if __name__ == "__main__":
    sys.exit(main())
