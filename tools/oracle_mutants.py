"""Mutation check of the oracle's geometry pins (tests/test_oracle_brute.py).

Copies oracle/, synthetic/ and tests/ to a scratch directory, applies one plausible
mistake at a time to oracle/sipg.py and runs the brute-force pins against it.  Every
mutant must make at least one pin fail; the unmutated copy must pass.

    python tools/oracle_mutants.py
"""
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (name, old text, new text) in oracle/sipg.py
MUTANTS = [
    ("cell metric J^-1 <-> J^-T (first factor)",
     'gphys = np.einsum("cqkm,cqkr->cqmr", Jinv, gref)', 'gphys = np.einsum("cqmk,cqkr->cqmr", Jinv, gref)'),
    ("cell metric J^-1 <-> J^-T (second factor)",
     't = np.einsum("cqmk,cqkr->cqmr", Jinv, gphys)', 't = np.einsum("cqkm,cqkr->cqmr", Jinv, gphys)'),
    ("face normal from J^-1 e_d instead of J^-T e_d",
     "JiT_ed = Jinv[..., d, :]", "JiT_ed = Jinv[..., :, d]"),
    ("face gradient J^-1 instead of J^-T",
     'gm = np.einsum("cfkm,cfkr->cfmr", Jinv_m, grm)', 'gm = np.einsum("cfmk,cfkr->cfmr", Jinv_m, grm)'),
    ("test-gradient term with J^-T n instead of J^-1 n",
     'cvec = np.einsum("cfmk,cfk->cfm", Jinv_m, nvec)', 'cvec = np.einsum("cfkm,cfk->cfm", Jinv_m, nvec)'),
    ("penalty max instead of mean",
     "sig_int = 0.5 * (AF / V + AFp / Vp)", "sig_int = np.maximum(AF / V, AFp / Vp)"),
    ("dropped symmetry (test-gradient) term",
     "rg = -0.5 * (dA[..., None] * jump)", "rg = -0.0 * (dA[..., None] * jump)"),
    ("wrong sign of the outward normal",
     "nvec = (2 * s - 1) * JiT_ed / nrm[..., None]", "nvec = (1 - 2 * s) * JiT_ed / nrm[..., None]"),
]


def run(tmp):
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
                        os.path.join(tmp, "tests", "test_oracle_brute.py")],
                       cwd=tmp, capture_output=True, text=True)
    return r.returncode, r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-200:]


def main():
    ok = True
    with tempfile.TemporaryDirectory() as tmp:
        for d in ("oracle", "synthetic", "tests"):
            shutil.copytree(os.path.join(ROOT, d), os.path.join(tmp, d),
                            ignore=shutil.ignore_patterns("__pycache__"))
        shutil.copy(os.path.join(ROOT, "pytest.ini"), tmp)
        src = os.path.join(tmp, "oracle", "sipg.py")
        orig = open(src).read()
        rc, tail = run(tmp)
        print(f"unmutated: rc={rc} {tail}")
        ok &= rc == 0
        for name, old, new in MUTANTS:
            assert old in orig, f"mutation site not found: {old}"
            open(src, "w").write(orig.replace(old, new))
            rc, tail = run(tmp)
            killed = rc != 0
            ok &= killed
            print(f"{'KILLED' if killed else 'SURVIVED'}: {name}: {tail}")
            open(src, "w").write(orig)
    print("all mutants killed" if ok else "SOME MUTANT SURVIVED")
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
