"""Golden convergence-study rows from the REFERENCE (acceptance.cpp criterion 4
settings: adv3d, nominal CFL steps, P2/P3, uniform/nonuniform), written to
tests/golden/acceptance_ref.json. Compiles a 20-line driver against the
unmodified reference headers (needs /root/reference; this container only).

    python tests/golden/make_acceptance_golden.py [meshes...]   (default 8 16 32)
"""
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REF_INC = os.environ.get("REF_INC", "/root/reference/proj/include")
DRIVER = r'''
#include "hgks/hgks.hpp"
#include <cstdio>
#include <cstdlib>
using namespace hgks;
int main(int argc, char** argv) {
    StudyOptions so;
    so.degree = std::atoi(argv[1]);
    so.nonuniform = std::atoi(argv[2]) != 0;
    so.nominal = true;
    so.workers = std::atoi(argv[3]);
    std::vector<int> meshes;
    for (int i = 4; i < argc; ++i) meshes.push_back(std::atoi(argv[i]));
    for (const auto& r : convergence_study("adv3d", meshes, so))
        std::printf("%d %.17g %.17g %.17g %d\n", r.n, r.err.l1, r.err.l2, r.err.cell_avg, r.steps);
}
'''


def main():
    meshes = [int(a) for a in sys.argv[1:]] or [8, 16, 32]
    exe = "/tmp/hgks_ref_study"
    with open(exe + ".cpp", "w") as f:
        f.write(DRIVER)
    subprocess.run(["g++", "-std=c++20", "-O3", "-march=native", "-pthread", "-I", REF_INC, exe + ".cpp", "-o", exe],
                   check=True)
    out = {}
    path = os.path.join(HERE, "acceptance_ref.json")
    if os.path.exists(path):
        out = json.load(open(path))
    degrees = [int(d) for d in os.environ.get("HGKS_DEGREES", "2 3").split()]
    for degree in degrees:
        for nonuni in (0, 1):
            key = f"adv3d_p{degree}_{'nonuniform' if nonuni else 'uniform'}"
            r = subprocess.run([exe, str(degree), str(nonuni), str(os.cpu_count()), *map(str, meshes)],
                               capture_output=True, text=True, check=True)
            rows = []
            for line in r.stdout.split("\n"):
                if line.strip():
                    n, l1, l2, ec, steps = line.split()
                    rows.append({"n": int(n), "l1": float(l1), "l2": float(l2), "cell_avg": float(ec),
                                 "steps": int(steps)})
            out[key] = rows
            json.dump(out, open(path, "w"), indent=1)
            print(key, rows, flush=True)


if __name__ == "__main__":
    main()
