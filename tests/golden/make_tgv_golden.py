"""Golden TGV P2 16^3 series (t <= 5, records every 0.05) and a final-state
digest from the REFERENCE (oracle/_ref), for tests/test_gpu_acceptance.py.
Needs the reference build (this container); ~3 min on 4 cores.

    python tests/golden/make_tgv_golden.py
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle as O  # noqa: E402


def main():
    r = O.RefRun("tgv", 16, 2, workers=os.cpu_count())
    steps, rec = r.advance(5.0, cfl=0.15, record_interval=0.05)
    q = r.get_state()[0].reshape(-1, 10, 5)
    out = {"case": "tgv", "n": 16, "degree": 2, "cfl": 0.15, "record_interval": 0.05, "t_end": 5.0,
           "steps": steps, "records_t_Ek_epsEk_epsZeta": rec.tolist(),
           "final_state": {"per_comp_l2": [float(np.sqrt(np.sum(q[:, n, v] ** 2))) for n in range(10)
                                           for v in range(5)], "max_abs": float(np.max(np.abs(q)))},
           "source": "reference headers compiled unmodified (oracle/_ref/libhgks_ref.so), RefRun.advance"}
    json.dump(out, open(os.path.join(HERE, "tgv16_ref.json"), "w"))


if __name__ == "__main__":
    main()
