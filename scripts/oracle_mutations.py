"""Mutation check of the oracle pins (CPU): apply one plausible mistake at a
time to oracle/hjcd_oracle.cpp, rebuild, run the CPU pins, and report which
test fails.  Every mutation must be caught.  The source is restored at the end.

    python scripts/oracle_mutations.py > profiles/r02a_oracle_mutations.log
"""
import os
import re
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "hjcd_oracle.cpp")

MUTATIONS = [
    ("W uses 1/(1 + |J_row|^2) (R17)", "(1.0 + std::sqrt(s))", "(1.0 + s)"),
    ("W drops w_o (R17)", "W[i] = (i < 3 ? c.w_p : c.w_o)", "W[i] = (i < 3 ? c.w_p : c.w_p)"),
    ("same joint keeps the SMALLER step (P:201, R8)",
     "bool take_p = std::fabs(dp[jp]) >= std::fabs(dor[jo]);",
     "bool take_p = std::fabs(dp[jp]) <= std::fabs(dor[jo]);"),
    ("gamma test on the squared change (literal Alg. 3 l.11, R10)",
     "double ip = e.ep - eh.ep, io = e.eo - eh.eo;",
     "double ip = (e.ep - eh.ep) * (e.ep - eh.ep), io = (e.eo - eh.eo) * (e.eo - eh.eo);"),
    ("gamma test: both spaces must improve (R10)", "bool accept = ap || ao;", "bool accept = ap && ao;"),
    ("position argmin takes the largest score (Alg. 3 l.9)", "if (sp[j] < sp[jp]) jp = j;", "if (sp[j] > sp[jp]) jp = j;"),
    ("dogleg accepted on |W rho| instead of |rho| (R23)",
     "double n0 = norm6(rho), nt = norm6(rt);\n        po.margin",
     "double n0 = std::sqrt(2 * cost_w(W, rho)), nt = std::sqrt(2 * cost_w(W, rt));\n        po.margin"),
    ("single coordinate takes argmin |g| (R24)",
     "        if (std::fabs(g[a]) > std::fabs(g[ist])) ist = a;\n    if (gap) {",
     "        if (std::fabs(g[a]) < std::fabs(g[ist])) ist = a;\n    if (gap) {"),
    ("dogleg tried before the LM step (Alg. 4 order)",
     "    bool ok = lm_step(c, J.data(), n, W, rho, dth.data());\n    if (ok) {",
     "    bool ok = lm_step(c, J.data(), n, W, rho, dth.data()) && false;\n    if (ok) {"),
    ("trust region not applied to the LM step (Alg. 4 l.6)",
     "for (int j = 0; j < n; ++j) dth[j] = clampd(dth[j], -c.R, c.R); /* l.6, R21 */", ""),
    ("Box-Muller pairs (u0,u2) instead of (u0,u1)", "double ua = u[2 * pair], ub = u[2 * pair + 1];",
     "double ua = u[pair], ub = u[pair + 2];"),
]


def main():
    orig = open(SRC).read()
    bak = SRC + ".bak"
    shutil.copy(SRC, bak)
    failed_to_catch = []
    try:
        for name, a, b in MUTATIONS:
            assert orig.count(a) == 1, f"pattern not unique: {name}"
            open(SRC, "w").write(orig.replace(a, b))
            r = subprocess.run([sys.executable, "-c", "import oracle; oracle.build(force=True)"], cwd=ROOT,
                               capture_output=True, text=True)
            if r.returncode:
                print(f"{name}: BUILD FAILED\n{r.stderr}")
                failed_to_catch.append(name)
                continue
            r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                                "tests/test_oracle_pins.py", "tests/test_oracle_pins_steps.py"],
                               cwd=ROOT, capture_output=True, text=True)
            fails = re.findall(r"^FAILED (\S+)", r.stdout, re.M)
            caught = r.returncode != 0
            print(f"{'caught' if caught else 'MISSED'}: {name} -> {fails[0] if fails else '-'}", flush=True)
            if not caught:
                failed_to_catch.append(name)
    finally:
        shutil.copy(bak, SRC)
        os.remove(bak)
        subprocess.run([sys.executable, "-c", "import oracle; oracle.build(force=True)"], cwd=ROOT)
    print(f"{len(MUTATIONS) - len(failed_to_catch)} / {len(MUTATIONS)} mutations caught")
    sys.exit(1 if failed_to_catch else 0)


if __name__ == "__main__":
    main()
