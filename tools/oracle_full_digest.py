"""Full-size parity pin: close a BASELINE config at its
full n with the CPU oracle's cache-blocked restatement and record the sha256
of the result (plus per-band digests, so a mismatch can be localised).

    python tools/oracle_full_digest.py c5_fw_u16 [--n 32768] [--threads 6]

Test infrastructure: runs in the build container (CPU only, ~10 min at
n = 32768 on 6 cores); the digest is committed to
tests/golden/config_digests.json and checked on the GPU by
tests/test_gpu_parity.py::test_c5_full_size_matches_oracle_digest.
"""
import argparse
import hashlib
import json
import sys
import time
from pathlib import Path

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))

import oracle  # noqa: E402
from paper_1705_08743_b200 import workloads  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--band", type=int, default=4096)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    cfg = workloads.CONFIGS[a.config]
    n = a.n or cfg.n
    (t,) = workloads.make_inputs(cfg, n)
    in_sha = hashlib.sha256(t.tobytes()).hexdigest()
    t0 = time.time()
    out = oracle.semiring_close_blocked(t, cfg.width, "anti", threads=a.threads)
    secs = time.time() - t0
    rec = {
        "config": cfg.name, "n": n, "seed": cfg.seed, "op": cfg.op, "width": cfg.width,
        "input_sha256": [in_sha],
        "output_sha256": hashlib.sha256(out.tobytes()).hexdigest(),
        "output_nonzero": int((out != 0).sum()),
        "band_rows": a.band,
        "band_sha256": [hashlib.sha256(out[r:r + a.band].tobytes()).hexdigest()
                        for r in range(0, n, a.band)],
        "source": "oracle (cache-blocked C restatement, oracle/semimat_oracle.c "
                  "DEFINE_CLOSE_BLOCKED; pinned to the reference's own C4 n=8192 sha256)",
        "oracle_seconds": round(secs, 1), "oracle_threads": a.threads or oracle.max_threads(),
        "layout": "padded lanes",
    }
    text = json.dumps(rec, indent=1)
    print(text)
    if a.out:
        Path(a.out).write_text(text + "\n")


if __name__ == "__main__":
    main()
