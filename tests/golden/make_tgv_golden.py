"""Golden TGV P2 series (records every 0.05) and a final-state digest from
the REFERENCE (oracle/_ref), for tests/test_gpu_acceptance.py and
tests/test_gpu_configs.py. Needs the reference build (this container).

    python tests/golden/make_tgv_golden.py            # 16^3 to t = 5  (~3 min, 4 cores)
    python tests/golden/make_tgv_golden.py 64 0.5     # BASELINE config C3 (~8 min, 8 cores)
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle as O  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    t_end = float(sys.argv[2]) if len(sys.argv) > 2 else 5.0
    r = O.RefRun("tgv", n, 2, workers=os.cpu_count())
    steps, rec = r.advance(t_end, cfl=0.15, record_interval=0.05)
    q = r.get_state()[0].reshape(-1, 10, 5)
    out = {"case": "tgv", "n": n, "degree": 2, "cfl": 0.15, "record_interval": 0.05, "t_end": t_end,
           "steps": steps, "records_t_Ek_epsEk_epsZeta": rec.tolist(),
           "final_state": {"per_comp_l2": [float(np.sqrt(np.sum(q[:, n, v] ** 2))) for n in range(10)
                                           for v in range(5)], "max_abs": float(np.max(np.abs(q)))},
           "source": "reference headers compiled unmodified (oracle/_ref/libhgks_ref.so), RefRun.advance"}
    json.dump(out, open(os.path.join(HERE, f"tgv{n}_ref.json"), "w"))


if __name__ == "__main__":
    main()
