"""bench.py -- decode/encode Msubpixel/s of the LPIC hot path on B200.

Default workload = BASELINE.json configs[1]: 24 synthetic 1/f RGB images of
768x512 per GPU (SURVEY 8(d) generator, seeds rank*24+k), the reference
network config (K=3, C=128, L=5, h=2) with "Kaiming seed 0" weights,
wavefront mode.

A step is one pass of the hot path over the batch: the wavefront decoder
over all payloads (the headline, `value`), and separately one encoder pass
(reported under "encode").  Device-resident timing uses CUDA events on the
launching stream around each step, with a 256 MiB L2 flush between steps
(outside the events); `e2e` times the public host-buffer C-ABI call
(lpic_decode_batch / lpic_encode_batch) including H2D and D2H copies.

Multi-GPU: one process per GPU.  `--gpus N` without a torchrun environment
re-launches itself under torch.distributed.run (127.0.0.1).  Images / tiles
are partitioned with paper_2212_01185_b200.shard (weak: every rank its own
images; strong: a fixed total split across ranks -- C3, C4, C5), no
collective on the data path; value = all ranks' sub-pixels / max-over-ranks
time (shard.reduce_over_ranks).  `--impl reference` times the reference
algorithm's CPU port (oracle/, the C restatement pinned to the reference's
golden vectors) on all host cores over a bounded sample of the same
workload, decode and encode.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FLOP_PER_SUBPX = 38912          # 58,368 MAC/px (network.py:145-156) * 2 / 3
CONFIGS = {
    "c2": dict(n=24, H=512, W=768, scaling="weak", desc="24 x 768x512 RGB per GPU (BASELINE configs[1])"),
    "c1": dict(n=1, H=64, W=64, kind="c1", scaling="weak",
               desc="1 x 64x64 RGB, 1/f seed 0 beta=2 sigma=3 (BASELINE configs[0])"),
    "c3": dict(n=256, H=1536, W=2048, scaling="strong", steps=1,
               desc="256 x 2048x1536 RGB sharded by image over the GPUs (BASELINE configs[2])"),
    "c3w": dict(n=32, H=1536, W=2048, scaling="weak",
                desc="32 x 2048x1536 RGB per GPU (= BASELINE configs[2]'s 256 at 8 GPUs)"),
    "c4": dict(n=256, H=512, W=512, kind="tiles", scaling="strong",
               desc="one 8192x8192 RGB image as 256 independently coded 512x512 tiles, sharded over GPUs "
                    "(BASELINE configs[3])"),
    "c5-1": dict(n=1, H=256, W=256, scaling="strong", desc="1 x 256x256 RGB (BASELINE configs[4])"),
    "c5-8": dict(n=8, H=256, W=256, scaling="strong", desc="8 x 256x256 RGB (BASELINE configs[4])"),
    "c5-64": dict(n=64, H=256, W=256, scaling="strong", desc="64 x 256x256 RGB (BASELINE configs[4])"),
    "c5-512": dict(n=512, H=256, W=256, scaling="strong", desc="512 x 256x256 RGB (BASELINE configs[4])"),
    "c5-4096": dict(n=4096, H=256, W=256, scaling="strong", desc="4096 x 256x256 RGB (BASELINE configs[4])"),
}

# DRAM bytes (read + write) per k_decode2 launch from one `ncu --set full`
# capture of the same workload (algorithmic: ~2 B per sub-pixel = image byte +
# payload; the rest is the L2-resident record ring spilling to DRAM)
NCU_TRAFFIC = {
    ("c2", "compat", False): (63398912 + 9401344, "profiles/r2/s3/ncu_r4f/dec_c2_raw_compact.csv"),
}
# measured on the box by scripts/ubench_phi_peak.cu / scripts/ubench_chain.cu
PEAKS_FILE = os.path.join(ROOT, "profiles", "r2", "ubench_peaks.json")
DEC_CLUSTER_SMS = 2             # k_decode2: one 2-CTA cluster per 1-2 streams


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def _synth_one(args):
    from paper_2212_01185_b200 import synth, tiles
    seed, H, W, gray = args
    if gray:
        return tiles.gray_to_rgb(synth.synth_1f_gray(seed, H, W))
    return synth.synth_1f(seed, H, W)


def make_images(cfgd, rank: int, world: int, gray: bool):
    """(images (n,H,W,3) u8) for this rank (shard.rank_units)."""
    from paper_2212_01185_b200 import shard, synth, tiles
    n, H, W = cfgd["n"], cfgd["H"], cfgd["W"]
    kind = cfgd.get("kind", "images")
    if kind == "c1":
        return np.stack([synth.c1_image()])
    if kind == "tiles":
        big = synth.synth_1f(0, 8192, 8192)
        grid = tiles.tile_grid(8192, 8192, H, W)
        lo, hi = shard.rank_units(len(grid), rank, world, "strong")
        return np.stack([big[i0:i0 + h, j0:j0 + w] for i0, j0, h, w in grid[lo:hi]]) if hi > lo else \
            np.zeros((0, H, W, 3), np.uint8)
    lo, hi = shard.rank_units(n, rank, world, cfgd["scaling"])
    jobs = [(s, H, W, gray) for s in range(lo, hi)]
    if not jobs:
        return np.zeros((0, H, W, 3), np.uint8)
    if len(jobs) * H * W >= (1 << 24):               # big batches: host processes in parallel
        from concurrent.futures import ProcessPoolExecutor
        with ProcessPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 1)) as ex:
            return np.stack(list(ex.map(_synth_one, jobs)))
    return np.stack([_synth_one(j) for j in jobs])


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback (B200_PROFILING.md)"


def load_ubench():
    if os.path.exists(PEAKS_FILE):
        with open(PEAKS_FILE) as f:
            return json.load(f)
    return {}


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
def _oracle_weights(w, cfg):
    from oracle import oracle as O
    return O.OracleWeights(w.tensors(), cfg.mixtures, cfg.filters, cfg.layers, cfg.kernel_half,
                           int(cfg.distribution))


def cpu_decode_sample(w, cfg, payloads, H, W, mode, threads, max_px):
    from oracle import oracle as O
    ow = _oracle_weights(w, cfg)
    streams = [payloads[k % len(payloads)] for k in range(threads)]
    t0 = time.perf_counter()
    O.decode_batch_prefix(ow, streams, H, W, mode, max_px, threads)
    dt = time.perf_counter() - t0
    return 3.0 * max_px * threads / dt / 1e6, dt


def cpu_encode_sample(w, cfg, imgs, mode, threads, max_px):
    from oracle import oracle as O
    ow = _oracle_weights(w, cfg)
    batch = np.stack([imgs[k % len(imgs)] for k in range(threads)])
    t0 = time.perf_counter()
    pays = O.encode_batch_prefix(ow, batch, mode, max_px, threads)
    dt = time.perf_counter() - t0
    return 3.0 * max_px * threads / dt / 1e6, dt, pays


def run_reference(args, cfgd):
    from paper_2212_01185_b200 import synth
    rank, world = env_int("RANK", 0), env_int("WORLD_SIZE", 1)
    if rank != 0:
        return
    w, cfg = synth.baseline_weights()
    if args.weights == "fitted":             # (the same fitted weights as our arm; fitting is not timed)
        w, cfg, _ = synth.fitted_weights()
    elif args.weights == "flat":
        w, cfg = synth.flat_weights()
    H, W = cfgd["H"], cfgd["W"]
    threads = os.cpu_count() or 1
    sub = dict(cfgd, n=min(cfgd["n"], threads), scaling="weak")
    imgs = make_images(sub, 0, 1, args.gray)[:threads]
    max_px = min(H * W, args.sample_px)
    # warm-up also produces the payloads the decode sample consumes
    payloads = None
    for _ in range(args.warmup):
        _, _, payloads = cpu_encode_sample(w, cfg, imgs, args.mode, threads, max_px)
        cpu_decode_sample(w, cfg, payloads, H, W, args.mode, threads, max_px)
    dec_t, enc_t = [], []
    for _ in range(args.steps):
        _, dt, payloads = cpu_encode_sample(w, cfg, imgs, args.mode, threads, max_px)
        enc_t.append(dt)
        dec_t.append(cpu_decode_sample(w, cfg, payloads, H, W, args.mode, threads, max_px)[1])
    subpx = 3.0 * max_px * threads
    value = subpx * args.steps / sum(dec_t) / 1e6
    enc_value = subpx * args.steps / sum(enc_t) / 1e6
    sample = (f"first {max_px} pixels (coding order) of {threads} concurrent {W}x{H} streams per step, "
              f"one stream per host thread (images reused cyclically if fewer)")
    line = {
        "metric": "decode Msubpixel/s (wavefront)", "value": value, "unit": "Msubpixel/s", "impl": "reference",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * sum(dec_t) / args.steps,
        "higher_is_better": True, "scaling": cfgd["scaling"], "vs_baseline": None, "dtype": "f32+f64",
        "data": "synthetic",
        "config": {"workload": cfgd["desc"], "mode": args.mode,
                   "weights": "kaiming seed 0" + (" fitted 200 steps" if args.weights == "fitted" else "")},
        "encode": {"value": enc_value, "unit": "Msubpixel/s", "ms_per_step": 1000.0 * sum(enc_t) / args.steps},
        "cpu_baseline": {"value": value, "unit": "Msubpixel/s", "cores": threads, "kind": "port",
                         "sample": sample, "encode_value": enc_value},
        "e2e": {"value": value, "unit": "Msubpixel/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def parity_check(w, cfg, imgs, pays, mode, threads):
    """Byte-compare GPU payloads with the C oracle's (pinned to the
    reference's golden vectors) on the given images; bpsp of both."""
    from oracle import oracle as O
    ow = _oracle_weights(w, cfg)
    t0 = time.perf_counter()
    ref = [O.encode(ow, np.ascontiguousarray(im), mode, threads=threads) for im in imgs]   # (threads within an image)
    dt = time.perf_counter() - t0
    same = sum(int(a == b) for a, b in zip(pays, ref))
    n_sub = 3.0 * imgs.shape[1] * imgs.shape[2] * len(ref)
    b_gpu = 8.0 * sum(len(p) for p in pays) / n_sub
    b_cpu = 8.0 * sum(len(p) for p in ref) / n_sub
    return {"images_checked": len(ref), "byte_identical": same, "bpsp_gpu": b_gpu, "bpsp_oracle": b_cpu,
            "bpsp_rel_delta": (b_gpu - b_cpu) / b_cpu, "oracle_s": dt,
            "note": "GPU containers vs the C oracle (pinned to the reference's own outputs, tests/golden)"}


def run_ours(args, cfgd):
    import torch
    import torch.distributed as dist

    import paper_2212_01185_b200 as P
    from paper_2212_01185_b200 import _native, shard, synth

    rank, world, local = env_int("RANK", 0), env_int("WORLD_SIZE", 1), env_int("LOCAL_RANK", 0)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", init_method="env://", device_id=dev)
    L = _native.require_cuda()
    w, cfg = synth.baseline_weights()
    fit_curve = None
    if args.weights == "fitted":
        w, cfg, fit_curve = synth.fitted_weights()
    elif args.weights == "flat":
        w, cfg = synth.flat_weights()
    H, W = cfgd["H"], cfgd["W"]
    N = H * W
    mode = P.parse_mode(args.mode)
    imgs = make_images(cfgd, rank, world, args.gray)
    n = imgs.shape[0]
    scaling = cfgd["scaling"]
    units_per_img = N if args.gray else 3 * N          # gray: one sample per pixel (r=g=b replicated)
    P.set_precision(args.precision)
    m = P.network.gpu_model(w, cfg)
    stream = torch.cuda.Stream(device=dev)
    sp = int(stream.cuda_stream)
    nn_ = max(n, 1)

    # resident inputs
    d_imgs = torch.from_numpy(imgs).to(dev) if n else torch.zeros((1, H, W, 3), dtype=torch.uint8, device=dev)
    cap_each = 6 * N + 64
    d_pay = torch.empty(nn_ * cap_each, dtype=torch.uint8, device=dev)
    d_lens = torch.zeros(nn_, dtype=torch.int64, device=dev)
    d_st = torch.zeros(nn_, dtype=torch.int32, device=dev)
    d_out = torch.empty((nn_, H, W, 3), dtype=torch.uint8, device=dev)
    d_offs = torch.arange(nn_, dtype=torch.int64, device=dev) * cap_each
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

    steps = args.steps
    # warm-up (also produces the payloads the decoder consumes)
    for _ in range(args.warmup):
        enc_dev()
        stream.synchronize()
    assert int(d_st[:n].sum().item()) == 0, "encoder status"
    lens = d_lens[:n].cpu().numpy()
    for _ in range(args.warmup):
        dec_dev()
        stream.synchronize()
    assert torch.equal(d_out[:n], d_imgs[:n]), "decoder is not lossless"

    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        dec_ms, dec_launch = timed(dec_dev, steps)
        enc_ms, enc_launch = timed(enc_dev, steps)
    torch.cuda.synchronize()
    assert torch.equal(d_out[:n], d_imgs[:n]), "decoder is not lossless"
    # the encoder's network stage on its own (K1 in SURVEY 2.2): compat = CUDA
    # cores in canonical fp32 order, fast = tcgen05 fp16x3 GEMMs
    net_n = min(n, 24)
    d_rawnet = torch.empty((max(net_n, 1), N, 12 * cfg.mixtures), dtype=torch.float32, device=dev)

    def net_dev():
        _native.check(L.lpic_network_coding_order(m.handle, d_imgs.data_ptr(), net_n, H, W, int(mode),
                                                   d_rawnet.data_ptr(), sp), "network")

    for _ in range(2):
        net_dev()
    stream.synchronize()
    net_ms, _ = timed(net_dev, steps)
    # the tcgen05 network (FAST precision, k_enc_net_tc2) on the same images,
    # so the default line carries the encoder's tensor-core fraction too
    tc_ms = None
    if args.precision == "compat" and n:
        P.set_precision("fast")
        try:
            mf = P.network.gpu_model(w, cfg)

            def tc_dev():
                _native.check(L.lpic_network_coding_order(mf.handle, d_imgs.data_ptr(), net_n, H, W, int(mode),
                                                           d_rawnet.data_ptr(), sp), "network (tcgen05)")

            for _ in range(2):
                tc_dev()
            stream.synchronize()
            tc_ms, _ = timed(tc_dev, steps)
        finally:
            P.set_precision("compat")
    del d_rawnet
    (t_dec, t_enc), units_all = shard.reduce_over_ranks([sum(dec_ms) / 1e3, sum(enc_ms) / 1e3],
                                                        float(units_per_img) * n, device=dev)
    dec_val = shard.aggregate_rate(units_all * steps, t_dec)
    enc_val = shard.aggregate_rate(units_all * steps, t_enc)

    # end to end through the public C-ABI with pinned host buffers
    h_img = torch.from_numpy(imgs).pin_memory() if n else torch.zeros(1, dtype=torch.uint8).pin_memory()
    h_pay = torch.empty(int(lens.sum()) + 64, dtype=torch.uint8).pin_memory()
    h_offs = np.zeros(nn_, np.int64)
    h_lens = np.zeros(nn_, np.int64)
    h_st = np.zeros(nn_, np.int32)
    h_out = torch.empty((nn_, H, W, 3), dtype=torch.uint8).pin_memory()

    def enc_e2e():
        _native.check(L.lpic_encode_batch(m.handle, h_img.data_ptr(), n, H, W, int(mode), h_pay.data_ptr(),
                                          h_pay.numel(), h_offs.ctypes.data, h_lens.ctypes.data, h_st.ctypes.data, sp),
                      "encode e2e")

    def dec_e2e():
        _native.check(L.lpic_decode_batch(m.handle, h_pay.data_ptr(), h_offs.ctypes.data, h_lens.ctypes.data, n, H, W,
                                          int(mode), h_out.data_ptr(), h_st.ctypes.data, sp), "decode e2e")

    enc_e2e()
    dec_e2e()                                   # (untimed warm-up of the host-buffer path)
    e2e_steps = max(1, min(steps, args.e2e_steps))
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        dec_e2e()
    e2e_dec_s = (time.perf_counter() - t0) / e2e_steps
    if n:
        assert torch.equal(h_out[:n], h_img), "e2e decode is not lossless"
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        enc_e2e()
    e2e_enc_s = (time.perf_counter() - t0) / e2e_steps
    (e2e_dec_max, e2e_enc_max), _ = shard.reduce_over_ranks([e2e_dec_s, e2e_enc_s], 0.0, device=dev)
    e2e_dec = shard.aggregate_rate(units_all, e2e_dec_max)
    e2e_enc = shard.aggregate_rate(units_all, e2e_enc_max)

    pays = [d_pay[b * cap_each:b * cap_each + int(lens[b])].cpu().numpy().tobytes() for b in range(n)]
    peaks, peak_kind = load_peaks()
    ub = load_ubench()
    dec_s_step = t_dec / steps
    bpsp = 8.0 * float(lens.sum()) / (float(units_per_img) * nn_)
    line = None
    if rank == 0:
        flop_unit = FLOP_PER_SUBPX * (3 if args.gray else 1)      # a gray pixel runs the net once for 3 sub-pixels
        achieved_tf = dec_val * 1e6 / world * flop_unit / 1e12
        metric = "decode Mpixel/s (grayscale, r=g=b)" if args.gray else "decode Msubpixel/s (wavefront)"
        unit = "Mpixel/s" if args.gray else "Msubpixel/s"
        subpx_local = 3.0 * N * n
        # per-GPU algorithmic DRAM bytes of one decode: payload read + image write
        alg_bytes = float(lens.sum()) + 3.0 * N * n
        phi_per_subpx = 255 * cfg.mixtures
        streams_per_cluster = 2 if n > 74 else 1
        clusters = (n + streams_per_cluster - 1) // streams_per_cluster
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        resident_streams = min(n, (sms // DEC_CLUSTER_SMS) * streams_per_cluster)
        line = {
            "metric": metric, "value": dec_val, "unit": unit, "n_gpus": world,
            "steps": steps, "warmup": args.warmup, "ms_per_step": 1000.0 * dec_s_step, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "f32+f64", "data": "synthetic",
            "config": {"workload": cfgd["desc"] + (" -- grayscale variant" if args.gray else ""),
                       "images_total": int(units_all / units_per_img), "images_rank0": n, "mode": args.mode,
                       "weights": ("kaiming seed 0 (K=3,C=128,L=5,h=2)" if args.weights == "kaiming" else
                                   "kaiming seed 0 with log-scale biases 7 (near-flat mixtures)" if args.weights == "flat"
                                   else "kaiming seed 0 fitted 200 steps on the GPU trainer (K=3,C=128,L=5,h=2), "
                                   f"final train loss {fit_curve[-1].loss_bits_per_pixel / 3:.3f} bpsp"),
                       "precision": ("compat (bit-exact fp32 net)" if args.precision == "compat"
                                     else "fast (tcgen05 fp16x3 net)"),
                       "l2": "256 MiB flush between timed steps",
                       "partition": f"{scaling}: shard.rank_units, no collective on the data path"},
            "encode": {"value": enc_val, "unit": unit, "ms_per_step": 1000.0 * t_enc / steps,
                       "e2e": e2e_enc, "gpu_launches": enc_launch},
            ("bits_per_gray_pixel" if args.gray else "bpsp"): bpsp,
            "e2e": {"value": e2e_dec, "unit": unit, "h2d_bytes_per_step": int(lens.sum()) + 16 * n,
                    "d2h_bytes_per_step": int(3 * N * n) + 4 * n},
            "roofline": {"bound": "tensor", "achieved": achieved_tf, "peak": peaks["bf16_tflops"],
                         "unit": "TFLOP/s", "frac": achieved_tf / peaks["bf16_tflops"],
                         "traffic": NCU_TRAFFIC.get((args.config, args.precision, args.gray), (None, None))[0],
                         "traffic_source": NCU_TRAFFIC.get((args.config, args.precision, args.gray), (None, None))[1],
                         "peak_kind": peak_kind,
                         "note": "model FLOPs (38,912/sub-pixel) per decode (SURVEY 8(d)); the decoder is bound by "
                                 "the serial per-stream range-coder chain -- see `chain`"},
            "hbm": {"achieved_gbs": alg_bytes / dec_s_step / 1e9, "peak_gbs": peaks["hbm_gbs"],
                    "frac": alg_bytes / dec_s_step / 1e9 / peaks["hbm_gbs"], "algorithmic_bytes_per_step": alg_bytes,
                    "note": "payload read + image write per decode, rank 0"},
            "phi": {"evals_per_s": dec_val * 1e6 / world * phi_per_subpx / (3 if args.gray else 1),
                    "per_subpixel": phi_per_subpx},
            "occupancy": {"streams_per_cluster": streams_per_cluster, "clusters": clusters,
                          "ctas": 2 * clusters, "sms": sms,
                          "sm_fraction": min(1.0, 2.0 * clusters / sms),
                          "threads_per_cta": 256 if streams_per_cluster == 1 else 384},
            "gpu_launches": dec_launch,
            "clocks": clk.summary(),
        }
        if ub.get("phi64_evals_per_s"):
            line["phi"]["peak"] = ub["phi64_evals_per_s"]
            line["phi"]["frac"] = line["phi"]["evals_per_s"] / ub["phi64_evals_per_s"]
            line["phi"]["peak_source"] = os.path.relpath(PEAKS_FILE, ROOT)
        if ub.get("chain_table_cycles"):
            clk_mhz = line["clocks"]["sm_mhz"] or 1965
            t_px = (2 * ub["chain_table_cycles"] + ub.get("chain_red_cycles", 400)) / (clk_mhz * 1e6)
            bound = resident_streams * 3.0 / t_px / 1e6
            line["chain"] = {"bound": bound, "frac": (dec_val / world) / bound, "unit": unit,
                             "t_pixel_us_isolated": t_px * 1e6, "resident_streams": resident_streams,
                             "formula": "resident streams x 3 / (2 t_table + t_red) at the sampled SM clock "
                                        "(isolated chain, scripts/ubench_chain.cu)"}
        net_s = sum(net_ms) / len(net_ms) / 1e3
        line["encode_network"] = {
            "kernel": "k_enc_net_tc2 (tcgen05)" if args.precision == "fast" else "k_enc_net (CUDA cores)",
            "images": net_n, "ms": net_s * 1e3,
            "model_tflops": 2.0 * 58368 * N * net_n / net_s / 1e12,
            "frac_of_bf16_peak": 2.0 * 58368 * N * net_n / net_s / 1e12 / peaks["bf16_tflops"],
            "note": ("model FLOPs (58,368 MAC/px); the fp16x3 split issues 3 MMAs per product and pads K 36->48, "
                     "N 36->48") if args.precision == "fast" else
                    "model FLOPs; canonical fp32 order (no FMA) cannot use tensor cores"}
        # the encoder's table stage (k_enc_tables + the fused range-coder plan,
        # plus the ~2 ms of k_rc_chunks / k_rc_merge): encode step minus the
        # network stage timed alone on the same images; its Phi rate against
        # the measured Phi peak is the encoder's roofline (255 K Phi per sub-pixel)
        if net_n == n and n:
            tab_s = t_enc / steps - net_s if world == 1 else None
            if tab_s and tab_s > 0:
                phi_rate = 3.0 * N * n * phi_per_subpx / tab_s       # (gray: r = g = b, three tables a pixel)
                line["encode_tables"] = {"ms": tab_s * 1e3, "phi_evals_per_s": phi_rate,
                                         "phi_peak": ub.get("phi64_evals_per_s"),
                                         "phi_frac": (phi_rate / ub["phi64_evals_per_s"]) if ub.get("phi64_evals_per_s") else None,
                                         "note": "encode step - network stage (includes the ~2 ms range-coder kernels)"}
        if tc_ms:
            tc_s = sum(tc_ms) / len(tc_ms) / 1e3
            model_tf = 2.0 * 58368 * N * net_n / tc_s / 1e12
            # issued: K 36 -> 48 and N 36 -> 48 padding, three fp16 MMAs per product (hi.hi, hi.lo, lo.hi)
            issued_tf = 3 * 2.0 * 61440 * N * net_n / tc_s / 1e12
            line["encode_network_tcgen05"] = {
                "kernel": "k_enc_net_tc2 (FAST precision, tcgen05/TMEM)", "images": net_n, "ms": tc_s * 1e3,
                "model_tflops": model_tf, "frac_of_bf16_peak": model_tf / peaks["bf16_tflops"],
                "issued_tflops": issued_tf, "issued_frac": issued_tf / peaks["bf16_tflops"],
                "note": "same images as encode_network; model FLOPs 58,368 MAC/px, issued 3 x 61,440 MAC/px"}
        cpu_threads = os.cpu_count() or 1
        if args.parity_images > 0 and args.precision == "compat" and n:
            k = min(args.parity_images, n)
            sel = sorted({int(round(i * (n - 1) / max(k - 1, 1))) for i in range(k)})
            line["parity"] = parity_check(w, cfg, imgs[sel], [pays[i] for i in sel], args.mode, cpu_threads)
            line["parity"]["images"] = sel
        if world == 1 and not args.no_cpu_baseline and n:
            max_px = min(N, args.sample_px)
            val, dt = cpu_decode_sample(w, cfg, pays[:cpu_threads], H, W, args.mode, cpu_threads, max_px)
            eval_, edt, _ = cpu_encode_sample(w, cfg, imgs[:cpu_threads], args.mode, cpu_threads, max_px)
            line["cpu_baseline"] = {"value": val, "unit": "Msubpixel/s", "cores": cpu_threads, "kind": "port",
                                    "encode_value": eval_,
                                    "sample": f"decode (and encode) of the first {max_px} pixels (coding order) of "
                                              f"{cpu_threads} streams, one per host thread ({dt:.1f} s / {edt:.1f} s)"}
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if line is not None:
        print(json.dumps(line), flush=True)


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=list(CONFIGS))
    ap.add_argument("--mode", default="wave", choices=["seq", "wave", "diag"])
    ap.add_argument("--sample-px", type=int, default=12288)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--parity-images", type=int, default=2,
                    help="byte-compare this many GPU containers with the C oracle (0: skip)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--weights", default="kaiming", choices=["kaiming", "fitted", "flat"],
                    help="BASELINE configs[1]: Kaiming seed 0, optionally fitted for 200 trainer steps; "
                         "flat: log-scale biases at the e^7 clip (near-flat PMFs, the selection worst case)")
    ap.add_argument("--gray", action="store_true", help="grayscale variant (r=g=b replication, BASELINE configs[4])")
    ap.add_argument("--precision", default="compat", choices=["compat", "fast"],
                    help="compat: reference-exact fp32 network (default); fast: tcgen05 fp16x3 network")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    cfgd = CONFIGS[args.config]
    if args.steps is None:
        args.steps = cfgd.get("steps", 5)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch under torchrun (rank 0 prints the line)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))
    if args.impl == "reference":
        run_reference(args, cfgd)
    else:
        run_ours(args, cfgd)


if __name__ == "__main__":
    main()
