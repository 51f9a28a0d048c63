"""Mutation check of the oracle's pin suite (CPU).

Each mutant below is a plausible mistake in oracle/dsmc_oracle.c.  The script
builds every mutant into a temporary library, runs the `-m "not gpu"` oracle
tests against it (oracle.py honours DSMC_ORACLE_LIB) and reports whether at
least one test fails -- a surviving mutant is an unpinned behaviour.
usage: python tools/mutate_oracle.py [--quick]"""
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "dsmc_oracle.c")
TESTS = ["tests/test_oracle_physics.py", "tests/test_oracle_rng.py", "tests/test_oracle_pins.py"]

MUTANTS = [
    ("diffuse bounce re-flies the full dt", "    tau = tau - t;\n", "    tau = tau;\n"),
    ("orifice removal deleted", "        if (R->open_face[(size_t)k * p->ny + j]) return 1;\n", "\n"),
    ("effusive entry flies the full dt", "        tau = u_co(a[0]) * R->dt_f;\n", "        tau = R->dt_f;\n"),
    ("post-step majorant update deleted", "    if (sgmax > gm) *gmax_c = (float)sgmax;\n", "\n"),
    ("jackknife factor n/(n-1)", "o[5 + q] = sqrt((double)(n_runs - 1) / (double)n_runs * ss);",
     "o[5 + q] = sqrt((double)n_runs / (double)(n_runs - 1) * ss);"),
    ("periodic wrap off by one box", "      if (x[a] >= L) x[a] = x[a] - L;\n", "      if (x[a] > L) x[a] = x[a] - L;\n"),
    ("pair index j not shifted past i", "    if (j >= i) j++;\n", "    if (j > i) j++;\n"),
    ("HS acceptance without the square", "      accept = lhs * lhs < (double)g2;\n", "      accept = lhs < (double)g2;\n"),
    ("post-collision sign flipped", "vx[j] = cmx - h * e[0];", "vx[j] = cmx + h * e[0];"),
    ("N(N-1) -> N*N in the candidate count", "double x = ((double)((int64_t)N * (N - 1)) * 0.5) * R->coef * gm;",
     "double x = ((double)((int64_t)N * N) * 0.5) * R->coef * gm;"),
    ("fault latch first-wins", "if (fault_rank(code) > fault_rank(R->status)) R->status = code;",
     "if (R->status == 0) R->status = code;"),
    ("sampling sums before the energy square", "      se += (vx * vx + vy * vy) + vz * vz;\n", "      se += (vx + vy) + vz;\n"),
    ("indexing unstable (descending within a cell)",
     "  for (int64_t i = 0; i < R->n; i++) if (R->cell[i] >= 0) R->lcr[cursor[R->cell[i]]++] = i;",
     "  for (int64_t i = R->n - 1; i >= 0; i--) if (R->cell[i] >= 0) R->lcr[cursor[R->cell[i]]++] = i;"),
]


def main():
    src = open(SRC).read()
    survivors = []
    for name, old, new in MUTANTS:
        assert src.count(old) == 1, (name, src.count(old))
        with tempfile.TemporaryDirectory() as d:
            c = os.path.join(d, "m.c")
            so = os.path.join(d, "m.so")
            open(c, "w").write(src.replace(old, new))
            subprocess.check_call(["gcc", "-O2", "-std=gnu11", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
                                   "-shared", "-I", os.path.join(ROOT, "oracle"), "-o", so, c, "-lm"])
            env = dict(os.environ, DSMC_ORACLE_LIB=so)
            r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider", *TESTS],
                               cwd=ROOT, env=env, capture_output=True, text=True)
            caught = r.returncode != 0
            last = [l for l in r.stdout.splitlines() if l.startswith("FAILED")][:1]
            print(f"{'caught  ' if caught else 'SURVIVED'} {name}  {last[0][:110] if last else ''}", flush=True)
            if not caught:
                survivors.append(name)
    print(f"{len(MUTANTS) - len(survivors)}/{len(MUTANTS)} mutants caught")
    return 1 if survivors else 0


if __name__ == "__main__":
    sys.exit(main())
