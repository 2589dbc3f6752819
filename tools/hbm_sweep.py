"""HBM-bound kernels at working sets >= 4x L2: K1 returns (GAE/lambda-return,
V-trace) through the standalone `tlg_returns` C ABI, and K7 (Adam / SGD) from the
learner's own CUDA-event phase timer on a wide trunk with a tiny batch.

At the named configs both kernels are L2-resident and latency-bound; this sweep shows
the fraction of measured HBM bandwidth they reach once the data has to stream.

    python tools/hbm_sweep.py [--out gpurun_out/hbm_sweep.json]
"""
import argparse
import ctypes as C
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def peaks():
    p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                     "MEASURED_PEAKS.json")
    try:
        return json.load(open(p))["hbm_gbs"], "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 7700.0, "nominal fallback"


def sweep_returns(torch, reps=20, sizes=(4096, 65536, 524288, 1048576)):
    from paper_2011_12895_b200._capi import Hyper, check, lib
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(dev)
    out = []
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    for algo, name, b_frame in ((0, "ppo", 17), (1, "vtrace", 25)):
        for S in sizes:
            T = 32
            g = torch.Generator(device=dev).manual_seed(S + algo)
            r = torch.rand(S, T, device=dev, generator=g) * 2 - 1
            v = torch.rand(S, T, device=dev, generator=g) * 2 - 1
            d = (torch.rand(S, T, device=dev, generator=g) < 0.01).to(torch.uint8)
            boot = torch.rand(S, device=dev, generator=g)
            valid = torch.full((S,), T, dtype=torch.int32, device=dev)
            bl = torch.full((S, T), float(np.log(1 / 6)), device=dev)
            tl = bl + 0.1 * (torch.rand(S, T, device=dev, generator=g) * 2 - 1)
            adv = torch.empty(S, T, device=dev)
            tgt = torch.empty(S, T, device=dev)
            h = Hyper.make()
            args = (algo, C.byref(h), S, T, r.data_ptr(), v.data_ptr(), d.data_ptr(),
                    boot.data_ptr(), valid.data_ptr(), bl.data_ptr(), tl.data_ptr(),
                    adv.data_ptr(), tgt.data_ptr(), C.c_void_p(stream.cuda_stream))
            torch.cuda.synchronize()
            for _ in range(3):
                check(lib().tlg_returns(*args))
            ms = []
            for _ in range(reps):
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                check(lib().tlg_returns(*args))  # synchronises the stream itself
                e1.record(stream)
                e1.synchronize()
                ms.append(e0.elapsed_time(e1))
            ms = float(np.median(ms))
            F = S * T
            nbytes = F * b_frame + S * 8
            out.append(dict(kernel="K1 returns_kernel + finalize_adv_kernel", algo=name,
                            segments=S, unroll_len=T, frames=F, algorithmic_bytes=nbytes,
                            working_set_over_l2=round(nbytes / l2, 2), ms=ms,
                            gbs=nbytes / (ms * 1e-3) / 1e9,
                            note="median of %d tlg_returns calls (CUDA events on the call's "
                                 "stream; includes the call's own err-flag D2H)" % reps))
            del r, v, d, boot, valid, bl, tl, adv, tgt
    return out


def sweep_optimizer(torch, steps=10):
    import paper_2011_12895_b200 as tlg
    out = []
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    S, T, D, A, hidden = 8, 32, 64, 6, (2048,) * 8
    for opt, b_param in (("adam", 28), ("sgd", 12)):
        lrn = tlg.Learner("mlp", D, A, hidden, algo="ppo", optimizer=opt, max_segments=S,
                          unroll_len=T, device=0)
        lrn.set_hyper(learning_rate=1e-5, batch_size=S, unroll_len=T)
        lrn.set_params(tlg.synth.init_params_f32(lrn.n_params, 0.01, seed=5).astype(np.float64))
        b = tlg.synth.make_segments(S, T, D, A, seed=7)
        for _ in range(3):
            lrn.train_step(b)
        lrn.set_timing(True)
        ms = []
        for _ in range(steps):
            lrn.train_step(b)
            ms.append(float(lrn.phase_ms()[5]))
        lrn.set_timing(False)
        lrn.close()
        ms = float(np.median(ms))
        nbytes = lrn.n_params * b_param
        out.append(dict(kernel="K7 optimizer_guarded_kernel", optimizer=opt,
                        params=int(lrn.n_params), algorithmic_bytes=nbytes,
                        working_set_over_l2=round(nbytes / l2, 2), ms=ms,
                        gbs=nbytes / (ms * 1e-3) / 1e9,
                        note="MLP 64-2048x8, 8x32 frames; learner phase timer (CUDA events), "
                             "median of %d steps" % steps))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/hbm_sweep.json")
    ap.add_argument("--profile-returns", type=int, default=0,
                    help="only K1 at this many segments, 2 reps (for an ncu capture)")
    a = ap.parse_args()
    import torch
    if a.profile_returns:
        for r in sweep_returns(torch, reps=2, sizes=(a.profile_returns,)):
            print(r["algo"], r["ms"])
        return
    peak, src = peaks()
    rows = sweep_returns(torch) + sweep_optimizer(torch)
    for r in rows:
        r["frac_of_hbm_peak"] = r["gbs"] / peak
    res = dict(hbm_peak_gbs=peak, peak_source=src,
               l2_bytes=torch.cuda.get_device_properties(0).L2_cache_size, rows=rows)
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    json.dump(res, open(a.out, "w"), indent=1)
    for r in rows:
        print("%-40s %-7s ws/L2 %6.2f  %8.3f ms  %7.0f GB/s  %.2f" % (
            r["kernel"], r.get("algo", r.get("optimizer")), r["working_set_over_l2"], r["ms"],
            r["gbs"], r["frac_of_hbm_peak"]))


if __name__ == "__main__":
    main()
