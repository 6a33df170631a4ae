"""Mutation check of the oracle's pins ("What's missing" 1).

Applies one plausible mistake at a time to a COPY of oracle/locc_oracle.cpp, builds it under /tmp,
points the oracle binding at it (LOCC_ORACLE_LIB) and runs the CPU oracle pins.  A mutation that
leaves every pin green is a hole in the pins.  Prints one line per mutation; exits 1 on a survivor.

    python tools/oracle_mutations.py [pytest -k expression]
"""
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "locc_oracle.cpp")

ZB = "  static const float zb[512] = {0};\n"
MUTATIONS = {
    "enc.l2 ReLU dropped": [("dense(P.enc2, W.w2.data(), h1.data(), h2.data(), true, emul);",
                             "dense(P.enc2, W.w2.data(), h1.data(), h2.data(), false, emul);")],
    "enc.l3 ReLU dropped": [("dense(P.enc3, W.w3.data(), h2.data(), h3.data(), true, emul);",
                             "dense(P.enc3, W.w3.data(), h2.data(), h3.data(), false, emul);")],
    "obj.l1 ReLU dropped": [("dense(P.obj1, z.data(), a.data(), true);", "dense(P.obj1, z.data(), a.data(), false);")],
    "obj.l2 ReLU dropped": [("dense(P.obj2, a.data(), b.data(), true);", "dense(P.obj2, a.data(), b.data(), false);")],
    "obj.l3 ReLU dropped": [("dense(P.obj3, b.data(), u, true);", "dense(P.obj3, b.data(), u, false);")],
    "pair.l1 ReLU dropped": [("dense(P.pair1, v.data(), a.data(), true);", "dense(P.pair1, v.data(), a.data(), false);")],
    "pair.l2 ReLU dropped": [("dense(P.pair2, a.data(), b.data(), true);", "dense(P.pair2, a.data(), b.data(), false);")],
    "pair.l3 ReLU dropped": [("dense(P.pair3, b.data(), c.data(), true);", "dense(P.pair3, b.data(), c.data(), false);")],
    "U-Net skips c1<->c2": [("x = concat(d3, kU, c2, kU, n4);", "x = concat(d3, kU, c1, kU, n4);"),
                            ("x = concat(d2, kU, c1, kU, n4);", "x = concat(d2, kU, c2, kU, n4);")],
    "U-Net d3 skip from c2": [("x = concat(d4, kU, c3, kU, n4);", "x = concat(d4, kU, c2, kU, n4);")],
    "U-Net concat halves swapped": [("x = concat(d4, kU, c3, kU, n4);", "x = concat(c3, kU, d4, kU, n4);"),
                                    ("x = concat(d3, kU, c2, kU, n4);", "x = concat(c2, kU, d3, kU, n4);"),
                                    ("x = concat(d2, kU, c1, kU, n4);", "x = concat(c1, kU, d2, kU, n4);")],
}
for layer in ("enc2", "enc3", "obj1", "obj2", "obj3", "pair1", "pair2", "pair3"):
    MUTATIONS[f"{layer}.b zeroed"] = [("  p.out = take(1, kP);\n",
                                       f"  p.out = take(1, kP);\n{ZB}  p.{layer}.b = zb;\n")]


def main():
    kexpr = sys.argv[1] if len(sys.argv) > 1 else None
    src = open(SRC).read()
    survivors = []
    tmp = tempfile.mkdtemp(prefix="oracle_mut_")
    try:
        for name, edits in MUTATIONS.items():
            s = src
            for a, b in edits:
                assert s.count(a) == 1, (name, a)
                s = s.replace(a, b)
            d = os.path.join(tmp, name.replace(" ", "_").replace("<->", "-"))
            os.makedirs(d)
            shutil.copy(os.path.join(ROOT, "oracle", "locc_oracle.h"), d)
            open(os.path.join(d, "locc_oracle.cpp"), "w").write(s)
            so = os.path.join(d, "liblocc_oracle.so")
            subprocess.check_call(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-fPIC", "-pthread", "-shared",
                                   "-o", so, os.path.join(d, "locc_oracle.cpp")])
            env = dict(os.environ, LOCC_ORACLE_LIB=so)
            cmd = [sys.executable, "-m", "pytest", "-q", "-x", "-m", "not gpu", "-p", "no:cacheprovider",
                   "tests/test_oracle_pins.py", "tests/test_oracle_network.py", "tests/test_oracle_cells.py"]
            if kexpr:
                cmd += ["-k", kexpr]
            rc = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True).returncode
            print(f"{'KILLED  ' if rc else 'SURVIVED'} {name}", flush=True)
            if rc == 0:
                survivors.append(name)
    finally:
        shutil.rmtree(tmp, ignore_errors=True)
    print(f"{len(MUTATIONS) - len(survivors)}/{len(MUTATIONS)} mutations killed")
    sys.exit(1 if survivors else 0)


if __name__ == "__main__":
    main()
