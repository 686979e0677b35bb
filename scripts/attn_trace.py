"""Pipeline trace of the bf16 attention kernel (CTA 0), for tuning.

    AS_ATTN_TRACE=1 python scripts/attn_trace.py [--config c2] [--mode 0]

Events per CTA-local tile (clock64 cycles):
  0 producer: K slot free, issuing K      1 producer: V slot free, issuing V
  2 MMA: K landed (QK issued)             3 MMA: V landed
  4 MMA: P ready (PV issued)              5 softmax: S ready (start)
  6 softmax: P written (end)
"""
import argparse
import os
os.environ.setdefault("AS_DEBUG_LIB", "1")  # debug build: experiment switches / instruments
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("AS_ATTN_TRACE", "1")
import bench  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--ghz", type=float, default=1.965)
args = ap.parse_args()
# calibration: HBM copy bandwidth on this box right now (read+write bytes)
_a = torch.empty(1 << 29, dtype=torch.bfloat16, device="cuda")
_b = torch.empty_like(_a)
for _ in range(3):
    _b.copy_(_a)
_s, _e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
_s.record()
for _ in range(5):
    _b.copy_(_a)
_e.record()
torch.cuda.synchronize()
print(f"calibration: torch copy {2 * _a.numel() * 2 * 5 / (_s.elapsed_time(_e) / 1e3) / 1e9:.0f} GB/s")
del _a, _b
W = bench.make_workload(args.config, "cuda", world=int(os.environ.get("AS_BENCH_EMULATE_WORLD", "1")))
if os.environ.get("AS_TRACE_SCHEDULE"):
    W["schedule"] = W["ada"].parse_schedule(os.environ["AS_TRACE_SCHEDULE"])
for _ in range(3):
    bench.run_attention(W)
torch.cuda.synchronize()
W["ws_attn"].view[256:].zero_()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
bench.run_attention(W)
e.record()
torch.cuda.synchronize()
print(f"{args.config} mode={os.environ.get('AS_ATTN_DEBUG_MODE', '0')} attention {s.elapsed_time(e) * 1e3:.1f} us")
tr = W["ws_attn"].view[256:256 + 4096 * 64].view(torch.int64).cpu().numpy().reshape(4096, 8)
cta = tr[4096 - 512:].copy()
tr = tr[:4096 - 512]
cta = cta[cta[:, 0] != 0]
if len(cta):
    t0c = cta[:, 0].min()
    st = (cta[:, 0] - t0c) / 1e3
    en = (cta[:, 1] - t0c) / 1e3
    print(f"per-CTA timeline ({len(cta)} CTAs, us from first start):")
    print(f"  plan done median {np.median((cta[:, 2] - t0c) / 1e3):.2f}  max {((cta[:, 2] - t0c) / 1e3).max():.2f}")
    print(f"  start  median {np.median(st):.2f}  max {st.max():.2f}")
    print(f"  end    min {en.min():.2f}  p10 {np.percentile(en, 10):.2f}  median {np.median(en):.2f}  "
          f"p90 {np.percentile(en, 90):.2f}  max {en.max():.2f}")
    print(f"  busy fraction (sum of CTA spans / (CTAs x makespan)) {((en - st).sum() / (len(cta) * en.max())):.3f}")
    print("  end-time histogram (us):", np.histogram(en, bins=10)[0].tolist(), np.round(np.histogram(en, bins=10)[1], 1).tolist())
    if os.environ.get("AS_ATTN_DEBUG_MODE") == "6":  # prologue / plan sub-phases, per CTA from its own entry
        rel = lambda c: np.median((cta[:, c] - cta[:, 0]) / 1e3)
        print(f"  per CTA from entry (median us): loads+reductions {rel(5):.2f}, scans {rel(4):.2f}, "
              f"plan done {rel(2):.2f}, first S tile {rel(6):.2f}, O ready {rel(7):.2f}")
    tagged = cta[(cta[:, 3] >> 40) == 1]
    if len(tagged):
        smid = tagged[:, 3] & 0xFFFF
        nrec = (tagged[:, 3] >> 16) & 0xFFFF
        en_t = (tagged[:, 1] - t0c) / 1e3
        merged = tagged[:, 4] != 0
        print(f"  end: CTAs that merged a tail unit {en_t[merged].mean():.2f} us (n={merged.sum()}), "
              f"others {en_t[~merged].mean():.2f} (n={(~merged).sum()})")
        for nr in sorted(set(nrec.tolist())):
            m = nrec == nr
            print(f"  end with {nr} pieces: mean {en_t[m].mean():.2f} (n={m.sum()})")
        order = np.argsort(smid)
        # SM halves (die proxy): smid < 74 vs >= 74
        lo = smid < 74
        print(f"  end by smid half: <74 {en_t[lo].mean():.2f}  >=74 {en_t[~lo].mean():.2f}")
        per_sm = {}
        for s_, e_ in zip(smid.tolist(), en_t.tolist()):
            per_sm.setdefault(s_, []).append(e_)
        early = sorted(per_sm.items(), key=lambda kv: min(kv[1]))[:12]
        print("  earliest-finishing SMs (smid: ends):", [(k, [round(x, 1) for x in v]) for k, v in early])
    for col, nm in ((5, "partial written"), (4, "merge done")):
        sel = cta[cta[:, col] != 0]
        if len(sel):
            v = (sel[:, col] - t0c) / 1e3
            print(f"  {nm}: {len(sel)} CTAs, median {np.median(v):.2f} max {v.max():.2f} (us)")
    sp = cta[cta[:, 6] != 0]
    if len(sp):
        pw = (sp[:, 5] - t0c) / 1e3
        pub = (sp[:, 3] - t0c) / 1e3
        mg = (sp[:, 4] - t0c) / 1e3
        f6 = (sp[:, 6] - t0c) / 1e3
        o7 = (sp[:, 7] - t0c) / 1e3
        print(f"  split pieces: first S tile median {np.median(f6):.2f}; O ready median {np.median(o7):.2f}")
        if (sp[:, 5] != 0).any():
            print(f"  split pieces: partial written median {np.median(pw):.2f} max {pw.max():.2f}; all published median "
              f"{np.median(pub):.2f}; merge done median {np.median(mg):.2f} max {mg.max():.2f} (us)")
ep = tr[3000:3064].copy()
ep = ep[ep[:, 0] != 0]
if len(ep):
    print("CTA-0 epilogues (us rel. to last P written): O complete, O stored, partial visible, decided, done; flags(1 tail,2 merged,4 full)")
    for r_ in ep:
        rel_ = lambda e: round((r_[e] - r_[0]) / 1e3, 2) if r_[e] else None
        print("  ", rel_(1), rel_(2), rel_(3), rel_(4), rel_(5), int(r_[7]))
peer = tr[2500:3000].copy()
tr = tr[:2500]
n = int((tr[:, 0] != 0).sum())
tr = tr[:n].astype(np.float64)
t0 = tr[0, 0]
tr = (tr - t0) / args.ghz  # ns
# columns: 0 K issue, 1 V issue, 2 MMA: K landed, 3 MMA: V landed, 4 PV issue, 5 softmax start, 6 softmax end, 7 QK issue
ns = lambda x: f"{np.median(x):7.0f} (p10 {np.percentile(x, 10):6.0f}, p90 {np.percentile(x, 90):6.0f})"
print(f"tiles traced on CTA 0: {n}; span {tr[n - 1, 6]:.0f} ns; per tile {tr[n - 1, 6] / n:.0f} ns")
print("producer K issue interval     ", ns(np.diff(tr[:, 0])))
print("K issue -> K landed (MMA sees)", ns(tr[:, 2] - tr[:, 0]))
print("V issue -> V landed           ", ns(tr[:, 3] - tr[:, 1]))
print("K landed -> softmax start     ", ns(tr[:, 5] - tr[:, 2]))
print("softmax duration              ", ns(tr[:, 6] - tr[:, 5]))
print("P ready -> MMA sees P         ", ns(tr[:, 4] - tr[:, 6]))
print("V landed -> PV issue (wait P) ", ns(tr[:, 4] - tr[:, 3]))
print("producer waits for K slot: K issue minus PV of tile-4 issue", ns(tr[4:, 0] - tr[:-4, 4]))
np.set_printoptions(linewidth=200, suppress=True)
if os.environ.get("AS_ATTN_DEBUG_MODE") == "5":
    # softmax sub-stamps: 2 S loaded, 3 max done, 4 exp done, 7 P stored
    print("softmax: start->S loaded", ns(tr[:, 2] - tr[:, 5]), " ->max", ns(tr[:, 3] - tr[:, 2]),
          " ->exp", ns(tr[:, 4] - tr[:, 3]), " ->P stored", ns(tr[:, 7] - tr[:, 4]), " ->arrived", ns(tr[:, 6] - tr[:, 7]))
    pn2 = int((peer[:, 5] != 0).sum())
    if pn2 > 40:
        pr2 = peer[:pn2].astype(np.float64) / args.ghz
        print("peer:    start->S loaded", ns(pr2[:, 2] - pr2[:, 5]), " ->max", ns(pr2[:, 3] - pr2[:, 2]),
              " ->exp", ns(pr2[:, 4] - pr2[:, 3]), " ->P stored", ns(pr2[:, 7] - pr2[:, 4]), " ->arrived", ns(pr2[:, 6] - pr2[:, 7]))
print("QK issue -> softmax start      ", ns(tr[:, 5] - tr[:, 7]))
print("QK issue interval             ", ns(np.diff(tr[:, 7])))
print("cols: Kiss Viss Kland Vland PViss Sstart Send QKiss ; rows = tiles 20..36 (ns rel. to tile 20 K issue)")
if n > 20:
    print(np.round(tr[20:37, :8] - tr[20, 0]))
pn = int((peer[:, 5] != 0).sum())
if pn > 40:
    # peer CTA (pair mode): forward K / V times, softmax start / end, same clock base as CTA 0's tile 20 K issue
    pr = (peer[:pn].astype(np.float64) - t0) / args.ghz
    print("peer CTA 1 (pair): softmax start - leader softmax start", ns(pr[20:pn, 5] - tr[20:pn, 5]))
    print("peer CTA 1 (pair): softmax duration                    ", ns(pr[20:pn, 6] - pr[20:pn, 5]))
    print("peer CTA 1 (pair): softmax end - leader softmax end    ", ns(pr[20:pn, 6] - tr[20:pn, 6]))
    print("peer rows 20..30: Kfwd Vfwd Sstart Send (rel. leader tile 20 K issue)")
    print(np.round(pr[20:31][:, [0, 1, 5, 6]] - tr[20, 0]))
