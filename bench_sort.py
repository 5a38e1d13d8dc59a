"""Edge-output sort on one B200: 5-column edge records sorted
by source with the in-house radix sort (lc_sort_edges_device, csrc/sort.cu), device
resident, out of place.

    python bench_sort.py [--log2 24,26,28] [--keys a51|random64] [--reps 3]

Prints one JSON line per size: time per sort, records/s, and the HBM roofline of the
whole sort.  Algorithmic bytes per record: histogram + payload pack 72 (key and four
payload columns read, the 32-byte record-major payload written); the first pass 20 (key
in; key + row out); each further pass 24 (key + row in and out); the LSD route's last
pass 84 (key + row in, the record's 32-byte payload, five output columns); the MSD route
(from 2^16 records) adds the window histogram (8) and the group bounds (8) and ends with
the per-group sort (84, like the LSD last pass).  L2 is flushed before every
timed sort.  Parity: the output equals numpy's stable argsort order
(checked at the smallest size).
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--log2", default="24,26,28")
    ap.add_argument("--keys", default="a51", choices=["a51", "random64"])
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()

    import torch

    from paper_1210_6411_b200 import _native as N

    ctx = N.context(0)
    dev = torch.device("cuda", 0)
    st = torch.cuda.Stream(dev)
    torch.cuda.set_stream(st)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    hbm = float(peaks.get("hbm_gbs", 0)) * 1e9 or None
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for i, lg in enumerate(int(x) for x in args.log2.split(",")):
        n = 1 << lg
        g = torch.Generator(device=dev)
        g.manual_seed(lg)
        if args.keys == "a51":
            r1 = torch.randint(1, 1 << 19, (n,), device=dev, generator=g)
            r2 = torch.randint(1, 1 << 22, (n,), device=dev, generator=g)
            src = r1 | (r2 << 19) | (0x2AAA00 << 41)
            varying_bytes = 6  # bits 0..40 vary (R1, R2), bytes 6-7 hold R3 only
        else:
            src = torch.randint(-(1 << 63), (1 << 63) - 1, (n,), device=dev, generator=g, dtype=torch.int64)
            varying_bytes = 8
        cols = [src, torch.randint(0, 1 << 62, (n,), device=dev, generator=g), torch.arange(n, device=dev),
                torch.randint(0, 1000, (n,), device=dev, generator=g), torch.randint(0, 100, (n,), device=dev, generator=g)]
        outs = [torch.empty_like(c) for c in cols]
        pin = (C.c_void_p * 5)(*[c.data_ptr() for c in cols])
        pout = (C.c_void_p * 5)(*[c.data_ptr() for c in outs])

        def run():
            N.check(N.lib.lc_sort_edges_device(ctx.handle, n, pin, pout, C.c_void_p(st.cuda_stream)))

        run()
        torch.cuda.synchronize()
        parity = None
        if i == 0:
            h = [c.cpu().numpy().view(np.uint64) for c in cols]
            order = np.argsort(h[0], kind="stable")
            parity = all(bool((o.cpu().numpy().view(np.uint64) == c[order]).all()) for c, o in zip(h, outs))
        times = []
        for _ in range(args.reps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            run()
            e1.record(st)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1) / 1e3)
        s = min(times)
        # algorithmic bytes of the route the device picks (csrc/sort.cu): LSD below 2^16
        # records -- 72 (histogram + payload pack) + 20 (first pass) + 24 per further pass
        # + 84 (last pass, payload gather) -- else MSD: 72 + 8 (window histogram) + 20 + 24
        # per further window pass + 8 (group bounds) + 84 (per-group sort: key + row in,
        # key out, payload gathered and written)
        lg = (n - 1).bit_length()
        W = min(max(lg - 10, 8), 22) if n >= 1 << 16 and os.environ.get("LFSR_SORT_LSD") != "1" else 0
        if W:
            nd = (W + 7) // 8
            alg = n * (72 + 8 + 20 + 24 * (nd - 1) + 8 + 84)
        else:
            alg = n * (72 + 20 + 24 * (varying_bytes - 2) + 84)
        line = {"metric": "edge-output sort (5-column records by source)", "records": n, "keys": args.keys,
                "route": f"msd (window {W} bits)" if W else f"lsd ({varying_bytes} passes)",
                "seconds": s, "records_per_s": n / s,
                "roofline": {"bound": "hbm", "achieved": alg / s / 1e9, "peak": hbm / 1e9 if hbm else None,
                             "unit": "GB/s", "frac": alg / s / hbm if hbm else None,
                             "algorithmic_bytes_per_record": alg / n,
                             "peak_source": "MEASURED_PEAKS.json hbm_gbs"},
                "parity_vs_numpy_stable_argsort": parity}
        print(json.dumps(line), flush=True)
        del cols, outs, src
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
