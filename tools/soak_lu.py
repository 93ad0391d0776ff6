"""Determinism soak of the LU (shipped build): repeated getrf_ts / luc2 calls on the same matrices,
pivots and L compared bit for bit with the first call's (and getrf's pivots with luc2's).

  python tools/soak_lu.py [iterations]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2412_06551_b200 as rl  # noqa: E402
import synth  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 100
bad = 0
for (m, n, seed) in ((65536, 64, 21), (40000, 64, 3), (262144, 128, 5), (100000, 256, 9), (65536, 48, 21)):
    X = synth.baseline_matrix(m, n, 8, seed, device="cuda")
    cfg = rl.default_cfg(m, n)
    ref = None
    for it in range(iters):
        r = rl.luc2(X, cfg=cfg)
        piv, U, L11, L, info = rl.getrf_ts(X, cfg=cfg, want_L=True)
        cur = (r.piv.clone(), piv.clone(), L.clone())
        if ref is None:
            ref = cur
            if not torch.equal(cur[0], cur[1]):
                bad += 1
                print(f"{m}x{n}: luc2 pivots != getrf pivots on the first call")
        else:
            for name, a, b in zip(("luc2 piv", "getrf piv", "L"), ref, cur):
                if not torch.equal(a, b):
                    bad += 1
                    print(f"{m}x{n} it {it}: {name} differs from the first call")
    print(f"{m}x{n}: {iters} iterations done, mismatches so far {bad}", flush=True)
print("SOAK", "FAILED" if bad else "OK", bad)

# the whole pipelines: Q and R of repeated calls bit-equal to the first call's
for (algo, m, n, kw) in (("slhc3", 65536, 64, dict(s=128)), ("sslhc3", 1048576, 128, dict(s1=1024, s2=256)),
                         ("sslhc3", 262144, 256, dict(s1=2048, s2=512))):
    X = synth.baseline_matrix(m, n, 12, 4, device="cuda")
    ref = None
    for it in range(max(10, iters // 4)):
        r = getattr(rl, algo)(X, seed=4, **kw)
        cur = (r.Q.clone(), r.R.clone(), r.piv.clone())
        if ref is None:
            ref = cur
        elif not all(torch.equal(a, b) for a, b in zip(ref, cur)):
            bad += 1
            print(f"{algo} {m}x{n} it {it}: Q, R or piv differs from the first call")
    print(f"{algo} {m}x{n}: done, mismatches so far {bad}", flush=True)
print("SOAK(all)", "FAILED" if bad else "OK", bad)
