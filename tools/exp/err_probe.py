"""Worst output error (in units of the 2e-3 bf16 tolerance) of the
keys-on-lanes kernel vs the oracle on peaky / outlier / normal inputs at
M = 1, 8, 40, 72 (BMC_LIB selects the build)."""
import json
import os
import sys
sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
from harness import Pair  # noqa: E402
from paper_2511_12031_b200 import bmc, synth  # noqa: E402
bmc.load()
tag = sys.argv[1]
for variant in ("peaky", "outlier", "normal"):
    for H_kv, H_q, k in ((2, 2, 0), (2, 16, 0), (1, 8, 4), (1, 8, 8)):
        p = Pair(2, H_kv, H_q, 128, 64, 700, dtype="bf16", seed=29, variant=variant)
        p.gpu.set_option(bmc.BMC_OPT_ATTN_PATH, 4)
        for _ in range(3):
            p.append()
        it = 0
        while p.orc.stats()["valid_max"] < 650:
            p.append()
            k_adm = p.spec_write(k) if k else 0
            if it % 5 == 0:
                p.sdpa(n_valid=-1)
            if k_adm:
                if it % 5 != 0:
                    p.sdpa(n_valid=-1)
                p.commit_rows(synth.acceptance(31, it, 2, k_adm))
            it += 1
        M = H_q // H_kv * (1 + k)
        print(json.dumps({"lib": tag, "variant": variant, "M": M, "worst_x_tol": round(p.worst, 4)}),
              flush=True)
        p.close()
