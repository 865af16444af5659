"""Mutation check of the oracle's pins (run by hand, CPU only): each mutation of oracle/oracle.c
below must make tests/test_oracle_pins.py fail.  The original file is restored afterwards.

    python tools/oracle_mutations.py
"""
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "oracle.c")

MUTATIONS = {
    "naive >= instead of >": ("if (orc_dot(P + j * d, U + i * d, d) > g) ++c;", "if (orc_dot(P + j * d, U + i * d, d) >= g) ++c;"),
    "twophase >= instead of >": ("if (topvals[i * kk + t] > g) ++c;", "if (topvals[i * kk + t] >= g) ++c;"),
    "membership <= instead of <": ("member[qi * n + i] = (uint8_t)(c < k);\n        }\n    }\n}\n\n/* The same", "member[qi * n + i] = (uint8_t)(c <= k);\n        }\n    }\n}\n\n/* The same"),
    "scan tau <- 0 (P:481 as printed)": ("double tau = -INFINITY;\n    int64_t sc = 0;", "double tau = 0.0;\n    int64_t sc = 0;"),
    "margin: copies of q not excluded": ("if (memcmp(P + j * d, q, sizeof(float) * (size_t)d) == 0) continue;\n            double s", "double s"),
    "margin: no normalisation": ("mu[t] = (den > 0) ? (g - tau) / den : (g - tau);\n        free(top);", "mu[t] = (g - tau);\n        free(top);"),
    "sort: ties by descending id": ("return (a < b) ? -1 : (a > b);", "return (a > b) ? -1 : (a < b);"),
    "topk: ties keep the higher id": ("while (pos > 0 && s > v[pos - 1]) {", "while (pos > 0 && s >= v[pos - 1]) {"),
    "block bounds max instead of min": ("if (L[i * kk + j] < mn) mn = L[i * kk + j];", "if (L[i * kk + j] > mn || mn == INFINITY) mn = L[i * kk + j];"),
}


def main():
    orig = open(SRC).read()
    bak = tempfile.mktemp()
    shutil.copy(SRC, bak)
    ok = True
    try:
        for name, (a, b) in MUTATIONS.items():
            if a not in orig:
                print("%-40s NOT APPLICABLE (pattern missing)" % name)
                ok = False
                continue
            open(SRC, "w").write(orig.replace(a, b, 1))
            subprocess.run([sys.executable, "-c", "import oracle.oracle as o; o.build_oracle(True)"], cwd=ROOT,
                           check=True)
            r = subprocess.run([sys.executable, "-m", "pytest", "tests/test_oracle_pins.py", "-q", "-x"], cwd=ROOT,
                               capture_output=True, text=True)
            caught = r.returncode != 0
            ok &= caught
            print("%-40s %s" % (name, "caught" if caught else "NOT CAUGHT"))
    finally:
        shutil.copy(bak, SRC)
        subprocess.run([sys.executable, "-c", "import oracle.oracle as o; o.build_oracle(True)"], cwd=ROOT, check=True)
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
