"""bench.py -- decode/encode Msubpixel/s of the LPIC hot path on B200.

Default workload = BASELINE.json configs[1]: 24 synthetic 1/f RGB images of
768x512 (SURVEY 8(d) generator, seeds rank*24+k), the reference network
config (K=3, C=128, L=5, h=2) with "Kaiming seed 0" weights, wavefront mode.

A step is one pass of the hot path over the batch: the wavefront decoder
over all 24 payloads (the headline, `value`), and separately one encoder
pass (reported under "encode").  Device-resident timing uses CUDA events on
the launching stream around each step, with a 256 MiB L2 flush between
steps (outside the events); `e2e` times the public host-buffer C-ABI call
(lpic_decode_batch / lpic_encode_batch) including H2D and D2H copies.

Multi-GPU (torchrun): weak scaling, every rank decodes its own 24 images;
no collective on the data path; value = all ranks' sub-pixels / max-over-
ranks time.  `--impl reference` times the reference algorithm's CPU port
(oracle/, the C restatement pinned to the reference's golden vectors) on
all host cores over a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FLOP_PER_SUBPX = 38912          # 58,368 MAC/px (network.py:145-156) * 2 / 3
CONFIGS = {
    "c2": dict(n=24, H=512, W=768, desc="24 x 768x512 RGB (BASELINE configs[1])"),
    "c1": dict(n=1, H=64, W=64, kind="c1", desc="1 x 64x64 RGB, 1/f seed 0 beta=2 sigma=3 (BASELINE configs[0])"),
    "c3": dict(n=32, H=1536, W=2048, desc="32 x 2048x1536 RGB per GPU = 256 over 8 GPUs (BASELINE configs[2])"),
    "c4": dict(n=256, H=512, W=512, kind="tiles", scaling="strong",
               desc="one 8192x8192 RGB image as 256 independently coded 512x512 tiles, sharded over GPUs "
                    "(BASELINE configs[3])"),
    "c5-1": dict(n=1, H=256, W=256, desc="1 x 256x256 RGB (BASELINE configs[4])"),
    "c5-8": dict(n=8, H=256, W=256, desc="8 x 256x256 RGB (BASELINE configs[4])"),
    "c5-64": dict(n=64, H=256, W=256, desc="64 x 256x256 RGB (BASELINE configs[4])"),
    "c5-512": dict(n=512, H=256, W=256, desc="512 x 256x256 RGB (BASELINE configs[4])"),
    "c5-4096": dict(n=4096, H=256, W=256, desc="4096 x 256x256 RGB (BASELINE configs[4])"),
}


# DRAM bytes (read + write) per k_decode2 launch from one `ncu --set full`
# capture of the same workload (algorithmic: ~2 B per sub-pixel = image byte +
# payload; the rest is the L2-resident record ring spilling to DRAM)
NCU_TRAFFIC = {
    ("c2", "compat", False): (64194560 + 28143872, "profiles/r1_sweep3/ncu_dec_c2_raw.csv"),
}


def make_images(cfgd, rank: int, world: int, gray: bool):
    """(images (n,H,W,3) u8, description) for this rank.  Weak scaling: every
    rank codes its own images (seeds rank*n ...).  c4 (strong): one 8192^2
    image, this rank's contiguous share of its 256 tiles."""
    from paper_2212_01185_b200 import shard, synth, tiles
    n, H, W = cfgd["n"], cfgd["H"], cfgd["W"]
    kind = cfgd.get("kind", "images")
    if kind == "c1":
        return np.stack([synth.c1_image()])
    if kind == "tiles":
        big = synth.synth_1f(0, 8192, 8192)
        grid = tiles.tile_grid(8192, 8192, H, W)
        lo, hi = shard.shard_range(len(grid), rank, world)
        return np.stack([big[i0:i0 + h, j0:j0 + w] for i0, j0, h, w in grid[lo:hi]])
    if gray:
        return np.stack([tiles.gray_to_rgb(synth.synth_1f_gray(rank * n + k, H, W)) for k in range(n)])
    return synth.batch(n, H, W, seed0=rank * n)


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


class ClockSampler:
    """nvidia-smi-equivalent clocks/throttle sampling via NVML during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        except Exception as e:  # pragma: no cover
            self.error = str(e)
        return self

    def _run(self):
        nv = self._nv
        names = {
            getattr(nv, "nvmlClocksThrottleReasonHwSlowdown", 0x8): "hw_slowdown",
            getattr(nv, "nvmlClocksThrottleReasonHwThermalSlowdown", 0x40): "hw_thermal_slowdown",
            getattr(nv, "nvmlClocksThrottleReasonSwThermalSlowdown", 0x20): "sw_thermal_slowdown",
            getattr(nv, "nvmlClocksThrottleReasonSwPowerCap", 0x4): "sw_power_cap",
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self._h)
                for bit, nm in names.items():
                    if r & bit:
                        self.reasons.add(nm)
            except Exception:
                pass
            self._stop.wait(0.2)

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# reference arm: the reference algorithm's C port on all host cores
# ---------------------------------------------------------------------------
def cpu_sample(w, cfg, payloads, H, W, mode, threads, max_px):
    from oracle import oracle as O
    ow = O.OracleWeights(w.tensors(), cfg.mixtures, cfg.filters, cfg.layers, cfg.kernel_half, int(cfg.distribution))
    streams = [payloads[k % len(payloads)] for k in range(threads)]
    t0 = time.perf_counter()
    O.decode_batch_prefix(ow, streams, H, W, mode, max_px, threads)
    dt = time.perf_counter() - t0
    return 3.0 * max_px * threads / dt / 1e6, dt


def oracle_payloads(w, cfg, imgs, mode, threads, max_px):
    from oracle import oracle as O
    ow = O.OracleWeights(w.tensors(), cfg.mixtures, cfg.filters, cfg.layers, cfg.kernel_half, int(cfg.distribution))
    return O.encode_batch_prefix(ow, imgs, mode, max_px, threads)


def run_reference(args, cfgd):
    from paper_2212_01185_b200 import synth
    rank, world = env_int("RANK", 0), env_int("WORLD_SIZE", 1)
    if rank != 0:
        return
    w, cfg = synth.baseline_weights()
    if args.weights == "fitted":             # (the same fitted weights as our arm; fitting is not timed)
        w, cfg, _ = synth.fitted_weights()
    n, H, W = cfgd["n"], cfgd["H"], cfgd["W"]
    threads = os.cpu_count() or 1
    imgs = make_images(cfgd, 0, 1, args.gray)[:threads]
    # payloads from the oracle encoder, sampled: encode only what we decode
    max_px = min(H * W, args.sample_px)
    payloads = oracle_payloads(w, cfg, imgs, args.mode, threads, max_px)
    for _ in range(args.warmup):
        cpu_sample(w, cfg, payloads, H, W, args.mode, threads, max_px)
    times = [cpu_sample(w, cfg, payloads, H, W, args.mode, threads, max_px)[1] for _ in range(args.steps)]
    tot = sum(times)
    value = 3.0 * max_px * threads * args.steps / tot / 1e6
    sample = (f"first {max_px} pixels (coding order) of {threads} concurrent {W}x{H} streams per step, "
              f"one stream per host thread (streams reused cyclically if fewer images)")
    line = {
        "metric": "decode Msubpixel/s (wavefront)", "value": value, "unit": "Msubpixel/s", "impl": "reference",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * tot / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32+f64",
        "data": "synthetic", "config": {"workload": cfgd["desc"], "mode": args.mode, "weights": "kaiming seed 0" + (" fitted 200 steps" if args.weights == "fitted" else "")},
        "cpu_baseline": {"value": value, "unit": "Msubpixel/s", "cores": threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": "Msubpixel/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args, cfgd):
    import torch
    import torch.distributed as dist

    import paper_2212_01185_b200 as P
    from paper_2212_01185_b200 import _native, synth

    rank, world, local = env_int("RANK", 0), env_int("WORLD_SIZE", 1), env_int("LOCAL_RANK", 0)
    if world > 1:
        dist.init_process_group("nccl", init_method="env://")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    L = _native.require_cuda()
    w, cfg = synth.baseline_weights()
    fit_curve = None
    if args.weights == "fitted":
        w, cfg, fit_curve = synth.fitted_weights()
    H, W = cfgd["H"], cfgd["W"]
    N = H * W
    mode = P.parse_mode(args.mode)
    imgs = make_images(cfgd, rank, world, args.gray)
    n = imgs.shape[0]
    strong = cfgd.get("scaling", "weak") == "strong"
    units_per_img = N if args.gray else 3 * N          # gray: one sample per pixel (r=g=b replicated)
    P.set_precision(args.precision)
    m = P.network.gpu_model(w, cfg)
    stream = torch.cuda.Stream(device=dev)
    sp = int(stream.cuda_stream)

    # resident inputs
    d_imgs = torch.from_numpy(imgs).to(dev)
    cap_each = 6 * N + 64
    d_pay = torch.empty(n * cap_each, dtype=torch.uint8, device=dev)
    d_lens = torch.zeros(n, dtype=torch.int64, device=dev)
    d_st = torch.zeros(n, dtype=torch.int32, device=dev)
    d_out = torch.empty((n, H, W, 3), dtype=torch.uint8, device=dev)
    d_offs = torch.arange(n, dtype=torch.int64, device=dev) * cap_each
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def enc_dev():
        _native.check(L.lpic_encode_batch_device(m.handle, d_imgs.data_ptr(), n, H, W, int(mode), d_pay.data_ptr(),
                                                 cap_each, d_lens.data_ptr(), d_st.data_ptr(), None, None, sp),
                      "encode")

    def dec_dev():
        _native.check(L.lpic_decode_batch_device(m.handle, d_pay.data_ptr(), d_offs.data_ptr(), d_lens.data_ptr(), n,
                                                 H, W, int(mode), d_out.data_ptr(), d_st.data_ptr(), None, None, sp),
                      "decode")

    def timed(fn, steps):
        ms = []
        launches = 0
        for _ in range(steps):
            with torch.cuda.stream(stream):
                flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            stream.synchronize()
            ms.append(e0.elapsed_time(e1))
            launches += int(L.lpic_last_launch_count(m.handle))
        return ms, launches

    # warm-up (also produces the payloads the decoder consumes)
    for _ in range(args.warmup):
        enc_dev()
        stream.synchronize()
    assert int(d_st.sum().item()) == 0
    lens = d_lens.cpu().numpy()
    for _ in range(args.warmup):
        dec_dev()
        stream.synchronize()
    assert torch.equal(d_out, d_imgs), "decoder is not lossless"

    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        dec_ms, dec_launch = timed(dec_dev, args.steps)
        enc_ms, enc_launch = timed(enc_dev, args.steps)
    torch.cuda.synchronize()
    assert torch.equal(d_out, d_imgs), "decoder is not lossless"
    # the encoder's network stage on its own (K1 in SURVEY 2.2): compat = CUDA
    # cores in canonical fp32 order, fast = tcgen05 fp16x3 GEMMs
    d_rawnet = torch.empty((n, N, 12 * cfg.mixtures), dtype=torch.float32, device=dev)

    def net_dev():
        _native.check(L.lpic_network_coding_order(m.handle, d_imgs.data_ptr(), n, H, W, int(mode),
                                                   d_rawnet.data_ptr(), sp), "network")

    for _ in range(2):
        net_dev()
    stream.synchronize()
    net_ms, _ = timed(net_dev, args.steps)
    del d_rawnet
    tot_dec = torch.tensor([sum(dec_ms)], dtype=torch.float64, device=dev)
    tot_enc = torch.tensor([sum(enc_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tot_dec, op=dist.ReduceOp.MAX)
        dist.all_reduce(tot_enc, op=dist.ReduceOp.MAX)
    n_all = torch.tensor([n], dtype=torch.int64, device=dev)
    if world > 1:
        dist.all_reduce(n_all, op=dist.ReduceOp.SUM)
    subpx = float(units_per_img) * int(n_all.item()) * args.steps
    dec_val = subpx / (tot_dec.item() / 1e3) / 1e6
    enc_val = subpx / (tot_enc.item() / 1e3) / 1e6

    # end to end through the public C-ABI with pinned host buffers
    h_img = torch.from_numpy(imgs).pin_memory()
    h_pay = torch.empty(int(lens.sum()) + 64, dtype=torch.uint8).pin_memory()
    h_offs = np.zeros(n, np.int64)
    h_lens = np.zeros(n, np.int64)
    h_st = np.zeros(n, np.int32)
    h_out = torch.empty((n, H, W, 3), dtype=torch.uint8).pin_memory()

    def enc_e2e():
        _native.check(L.lpic_encode_batch(m.handle, h_img.data_ptr(), n, H, W, int(mode), h_pay.data_ptr(),
                                          h_pay.numel(), h_offs.ctypes.data, h_lens.ctypes.data, h_st.ctypes.data, sp),
                      "encode e2e")

    def dec_e2e():
        _native.check(L.lpic_decode_batch(m.handle, h_pay.data_ptr(), h_offs.ctypes.data, h_lens.ctypes.data, n, H, W,
                                          int(mode), h_out.data_ptr(), h_st.ctypes.data, sp), "decode e2e")

    enc_e2e()
    dec_e2e()                                   # (untimed warm-up of the host-buffer path)
    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        dec_e2e()
    e2e_dec_s = (time.perf_counter() - t0) / e2e_steps
    assert torch.equal(h_out, h_img), "e2e decode is not lossless"
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        enc_e2e()
    e2e_enc_s = (time.perf_counter() - t0) / e2e_steps
    e2e = torch.tensor([e2e_dec_s, e2e_enc_s], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e, op=dist.ReduceOp.MAX)
    per_step_subpx = float(units_per_img) * int(n_all.item())
    e2e_dec = per_step_subpx / e2e[0].item() / 1e6
    e2e_enc = per_step_subpx / e2e[1].item() / 1e6

    peaks, peak_kind = load_peaks()
    dec_ms_step = tot_dec.item() / args.steps
    bpsp = 8.0 * float(lens.sum()) / (float(units_per_img) * n)
    line = None
    if rank == 0:
        flop_unit = FLOP_PER_SUBPX * (3 if args.gray else 1)      # a gray pixel runs the net once for 3 sub-pixels
        achieved_tf = dec_val * 1e6 / world * flop_unit / 1e12
        metric = "decode Mpixel/s (grayscale, r=g=b)" if args.gray else "decode Msubpixel/s (wavefront)"
        unit = "Mpixel/s" if args.gray else "Msubpixel/s"
        line = {
            "metric": metric, "value": dec_val, "unit": unit, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dec_ms_step, "higher_is_better": True,
            "scaling": "strong" if strong else "weak", "vs_baseline": None, "dtype": "f32+f64", "data": "synthetic",
            "config": {"workload": cfgd["desc"] + (" -- grayscale variant" if args.gray else ""),
                       "images_per_gpu": n, "mode": args.mode,
                       "weights": ("kaiming seed 0 (K=3,C=128,L=5,h=2)" if args.weights == "kaiming" else
                                   "kaiming seed 0 fitted 200 steps on the GPU trainer (K=3,C=128,L=5,h=2), "
                                   f"final train loss {fit_curve[-1].loss_bits_per_pixel / 3:.3f} bpsp"),
                       "precision": ("compat (bit-exact fp32 net)" if args.precision == "compat"
                                     else "fast (tcgen05 fp16x3 net)"),
                       "l2": "256 MiB flush between timed steps"},
            "encode": {"value": enc_val, "unit": unit, "ms_per_step": tot_enc.item() / args.steps,
                       "e2e": e2e_enc},
            ("bits_per_gray_pixel" if args.gray else "bpsp"): bpsp,
            "e2e": {"value": e2e_dec, "unit": unit, "h2d_bytes_per_step": int(lens.sum()) + 16 * n,
                    "d2h_bytes_per_step": int(3 * N * n) + 4 * n},
            "roofline": {"bound": "tensor", "achieved": achieved_tf, "peak": peaks["bf16_tflops"],
                         "unit": "TFLOP/s", "frac": achieved_tf / peaks["bf16_tflops"],
                         "traffic": NCU_TRAFFIC.get((args.config, args.precision, args.gray), (None, None))[0],
                         "traffic_source": NCU_TRAFFIC.get((args.config, args.precision, args.gray), (None, None))[1],
                         "peak_kind": peak_kind,
                         "note": "model FLOPs (38,912/sub-pixel) per decode; the decoder is bound by the serial "
                                 "per-stream range-coder chain, see DESIGN.md"},
            "encode_network": {
                "kernel": "k_enc_net_tc (tcgen05)" if args.precision == "fast" else "k_enc_net (CUDA cores)",
                "ms": sum(net_ms) / len(net_ms),
                "model_tflops": 2.0 * 58368 * N * n / (sum(net_ms) / len(net_ms) / 1e3) / 1e12,
                "frac_of_bf16_peak": 2.0 * 58368 * N * n / (sum(net_ms) / len(net_ms) / 1e3) / 1e12 / peaks["bf16_tflops"],
                "note": "model FLOPs (58,368 MAC/px); the fp16x3 split issues 3 MMAs per product "
                        "and pads K 36->48, N 36->48" if args.precision == "fast" else
                        "model FLOPs; canonical fp32 order (no FMA) cannot use tensor cores"},
            "gpu_launches": dec_launch,
            "clocks": clk.summary(),
        }
        if world == 1 and not args.no_cpu_baseline:
            cpu_threads = os.cpu_count() or 1
            ps = [d_pay[b * cap_each:b * cap_each + int(lens[b])].cpu().numpy().tobytes()
                  for b in range(min(n, cpu_threads))]
            max_px = min(N, args.sample_px)
            val, dt = cpu_sample(w, cfg, ps, H, W, args.mode, cpu_threads, max_px)
            line["cpu_baseline"] = {"value": val, "unit": "Msubpixel/s", "cores": cpu_threads, "kind": "port",
                                    "sample": f"decode of the first {max_px} pixels (coding order) of "
                                              f"{cpu_threads} GPU-encoded streams, one per host thread ({dt:.1f} s)"}
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if line is not None:
        print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=list(CONFIGS))
    ap.add_argument("--mode", default="wave", choices=["seq", "wave", "diag"])
    ap.add_argument("--sample-px", type=int, default=12288)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--weights", default="kaiming", choices=["kaiming", "fitted"],
                    help="BASELINE configs[1]: Kaiming seed 0, optionally fitted for 200 trainer steps")
    ap.add_argument("--gray", action="store_true", help="grayscale variant (r=g=b replication, BASELINE configs[4])")
    ap.add_argument("--precision", default="compat", choices=["compat", "fast"],
                    help="compat: reference-exact fp32 network (default); fast: tcgen05 fp16x3 network")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    cfgd = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfgd)
    else:
        run_ours(args, cfgd)


if __name__ == "__main__":
    main()
