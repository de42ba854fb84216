#!/usr/bin/env python3
"""Benchmark: autoregressive WaveNet sample generation (Deep Voice, arXiv 1702.07825).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload C2]

A *step* is one dvw_generate call: one whole utterance of the workload through
the full hot path (embedding, l gated dilated layers, skip/head, softmax,
inverse-CDF sampling, feedback), inputs resident in HBM.  The default workload
is BASELINE.json configs[1] = C2: l=20 r=64 s=256, batch 1, 16,000 samples
(1 s at 16 kHz), frame-rate conditioning with hop 64.  Under torchrun each rank
generates its own utterance (utterance id = rank): independent problems, no
collective on the data path, "scaling": "weak".  Rank 0 prints one JSON line.

--impl reference times the CPU oracle (oracle/, test infrastructure) on the
host cores, rank 0 only, each step a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1702_07825_b200 import synth  # noqa: E402

METRIC = "audio samples/sec per stream (batch-1 real-time factor at 16 kHz) and aggregate"
WORKLOADS = {
    "C1": dict(cfg=synth.C1, n=1600, streams=1, split=False,
               desc="C1: l=20 r=64 s=128, batch 1, 1,600 samples (0.1 s @16 kHz), hop 64"),
    "C2": dict(cfg=synth.C2, n=16000, streams=1, split=False,
               desc="C2: l=20 r=64 s=256, batch 1, 16,000 samples (1 s @16 kHz), hop 64"),
    "C3": dict(cfg=synth.C3, n=160000, streams=1, split=False,
               desc="C3: l=40 r=64 s=256, batch 1, 160,000 samples (10 s @16 kHz), hop 64"),
    # batched (tcgen05) workloads: streams per GPU (C4, weak) or in total, sharded (C5, strong)
    "C4": dict(cfg=synth.C4, n=80000, streams=256, split=False,
               desc="C4: l=20 r=128 s=256, 256 concurrent utterances per GPU batched (tcgen05), "
                    "80,000 samples (5 s @16 kHz) each, hop 64"),
    "C5": dict(cfg=synth.C5, n=80000, streams=2048, split=True,
               desc="C5: l=40 r=64 s=256, 2,048 utterances of 80,000 samples (5 s) sharded across "
                    "the GPUs (no collective on the path), batched (AUTO: tcgen05 batched kernel, or "
                    "streams interleaved on clusters below the measured crossover), hop 64"),
}
HOP = 64
FP32_FMA_PEAK_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12  # 74.4 TFLOP/s
TF32_RATIO = 0.5  # dense tf32 / bf16 tensor throughput (B200_PROFILING.md nominal 1.125 / 2.25 PFLOP/s)


def tf32_peak_tflops():
    """Dense tf32 peak = MEASURED_PEAKS.json sustained bf16 x the nominal tf32/bf16 ratio."""
    try:
        d = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return d["bf16_tflops_sustained"] * TF32_RATIO, "MEASURED_PEAKS.json bf16 sustained x 0.5"
    except Exception:
        return 1590.0 * TF32_RATIO, "B200_PROFILING.md fallback bf16 1.59 PFLOP/s x 0.5"


def hbm_peak_gbs():
    """Measured HBM copy bandwidth (MEASURED_PEAKS.json), else the guide's fallback."""
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"], "of measured"
    except Exception:
        return 6650.0, "of fallback (B200_PROFILING.md)"


def macs_per_sample(cfg) -> int:
    """l (5 r^2 + r s) + a s + a^2 (SURVEY.md §8(a) per-sample totals)."""
    L, r, s, a = cfg.n_layers, cfg.residual, cfg.skip, cfg.levels
    return L * (5 * r * r + r * s) + a * s + a * a


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """Samples SM clock + throttle reasons via NVML while the timed region runs."""

    def __init__(self, dev_index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(dev_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        names = {
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
            "hw_power_brake": getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                fn = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                    nv.nvmlDeviceGetCurrentClocksThrottleReasons
                mask = fn(self.h)
                for k, bit in names.items():
                    if mask & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            self._stop.wait(0.02)

    def __enter__(self):
        if self.nv is not None:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv is not None:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "n_samples": len(self.samples)}


def load_ncu_traffic(workload: str, stream_samples: int):
    """Per-launch DRAM bytes of the dominant kernel from the committed ncu summary
    (profiles/ncu_summary.json): the captured launch's bytes, or -- for the batched
    workloads, captured on a short launch -- bytes per stream-sample x this launch's
    stream-samples (the queue traffic scales with it)."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        d = json.load(open(p)).get(workload, {})
        if d.get("dram_bytes_per_launch") is not None:
            return d["dram_bytes_per_launch"]
        if d.get("dram_bytes_per_stream_sample") is not None:
            return d["dram_bytes_per_stream_sample"] * stream_samples
        return None
    except Exception:
        return None


def load_active_sm_pipes(workload: str):
    """FMA-pipe and shared-memory utilisation of the ACTIVE SMs of the batch-1 kernel, from the
    committed ncu capture (profiles/ncu_summary.json; the metrics are averaged over all 148 SMs
    there, so avg x 148 / active SMs is the active-SM mean)."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        d = json.load(open(p))[workload]
        a = d["active_sm_pipes"]
        return {"active_sms": a["active_sms"], "fma_pipe_pct_active_sms": a["fma_pct"],
                "smem_pct_active_sms": a["smem_pct"], "pipes_source": a["source"]}
    except Exception:
        return {}


def run_reference(args, wl):
    """The oracle (CPU, fp64, one core) on bounded samples of the workload."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    import oracle
    cfg, n_total = wl["cfg"], wl["n"]
    n = min(n_total, args.ref_samples)
    w = synth.make_weights(cfg, 0)
    cond = synth.make_cond(cfg, synth.n_frames_for(n_total, HOP), 0)
    u = synth.make_uniforms(n_total, 0)
    for _ in range(args.warmup if args.warmup <= 1 else 1):
        oracle.run(cfg.n_layers, cfg.residual, cfg.skip, w, cond, HOP, min(n, 64), uniforms=u,
                   dilations=cfg.dilation_list(), want_logits=False)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.run(cfg.n_layers, cfg.residual, cfg.skip, w, cond, HOP, n, uniforms=u,
                   dilations=cfg.dilation_list(), want_logits=False)
        times.append(time.perf_counter() - t0)
    sec = float(np.mean(times))
    value = n / sec
    sample = f"first {n} samples of the {args.workload} utterance (utterance 0), fp64 scalar C, 1 thread"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": wl["desc"], "samples_per_step": n, "streams": 1},
        "cpu_baseline": {"value": value, "unit": "samples/s", "cores": 1, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def cpu_baseline_and_parity(cfg, n, w, cond, u, gpu_codes, budget_samples, gpu_tf_logits=None, nonlin="exact"):
    """Oracle timed on this host (1 core) on the same utterance; plus parity on it
    (free-running codes, per-step mismatch rate, and -- when given -- the GPU's
    teacher-forced logits on its own codes against the oracle's)."""
    import oracle
    nb = min(n, budget_samples)
    t0 = time.perf_counter()
    ref_codes, _, _ = oracle.run(cfg.n_layers, cfg.residual, cfg.skip, w, cond, HOP, nb, uniforms=u[:nb],
                                 dilations=cfg.dilation_list(), want_logits=False, nonlin=nonlin)
    sec = time.perf_counter() - t0
    diff = np.nonzero(ref_codes != gpu_codes[:nb])[0]
    first = int(diff[0]) if diff.size else None
    # per-step mismatch rate: oracle teacher-forced on the GPU's own codes, drawing with the same u
    _, ref_lg, sampled = oracle.run(cfg.n_layers, cfg.residual, cfg.skip, w, cond, HOP, nb, uniforms=u[:nb],
                                    forced=gpu_codes[:nb], dilations=cfg.dilation_list(),
                                    want_logits=gpu_tf_logits is not None, want_sampled=True, nonlin=nonlin)
    mism = int(np.sum(sampled != gpu_codes[:nb]))
    cpu = {"value": nb / sec, "unit": "samples/s", "cores": 1, "kind": "oracle",
           "sample": f"{nb} samples of the same utterance (utterance 0), fp64 scalar C oracle, 1 thread"}
    parity = {"checked_samples": nb, "bit_exact_first_1600": bool(first is None or first >= 1600),
              "first_divergence": first, "divergence_rate": mism / nb, "mismatches": mism}
    if gpu_tf_logits is not None:
        k = min(nb, len(gpu_tf_logits))
        parity["teacher_forced_max_abs_dlogit"] = float(
            np.max(np.abs(gpu_tf_logits[:k].astype(np.float64) - ref_lg[:k])))
        parity["teacher_forced_samples"] = k
        parity["teacher_forced_gate"] = 1e-3
    return cpu, parity


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def cpu_c1_aggregate(n_samples=1600):
    """the oracle on C1 (l=20, r=64, s=128, 1,600 samples, utterance 0)
    on one thread, then K = len(os.sched_getaffinity(0)) independent C1 utterances (0..K-1) on K
    threads at once (the C oracle releases the GIL inside its ctypes call); aggregate samples/s."""
    import concurrent.futures as cf
    import oracle
    c1 = synth.Config(20, 64, 128)
    w = synth.make_weights(c1, 0)
    nf = (n_samples + HOP - 1) // HOP
    K = len(os.sched_getaffinity(0))
    inputs = [(synth.make_cond(c1, nf, u), synth.make_uniforms(n_samples, u)) for u in range(K)]

    def one(k):
        cond, u = inputs[k]
        t0 = time.perf_counter()
        oracle.run(c1.n_layers, c1.residual, c1.skip, w, cond, HOP, n_samples, uniforms=u,
                   dilations=c1.dilation_list(), want_logits=False)
        return time.perf_counter() - t0

    single = one(0)
    t0 = time.perf_counter()
    with cf.ThreadPoolExecutor(max_workers=K) as ex:
        list(ex.map(one, range(K)))
    wall = time.perf_counter() - t0
    return {"config": "C1 l=20 r=64 s=128, 1,600 samples per utterance (0.1 s at 16 kHz)",
            "single_thread_s": single, "single_thread_samples_per_s": n_samples / single,
            "threads": K, "aggregate_wall_s": wall, "aggregate_samples_per_s": K * n_samples / wall}


def device_inputs(cfg, n, utts, dev):
    """Batched workloads: conditioning U(-0.5, 0.5) and uniforms U[0, 1) drawn on the device,
    each element a counter-based hash of (role, utterance id, index) (synth.make_batch_hashed_torch;
    DESIGN.md "Input recipe"): an utterance's inputs do not depend on its batch, rank or the GPU
    count, so its codes are comparable across every G (host arrays of 2,048 x 5 s would not fit)."""
    return synth.make_batch_hashed_torch(cfg, n, utts, HOP, dev)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="C2", choices=sorted(WORKLOADS))
    ap.add_argument("--kernel", default="auto", choices=["auto", "cluster", "stream", "tc"])
    ap.add_argument("--precision", default="fp32", choices=["fp32", "tf32", "approx", "appc"],
                    help="tf32: one-pass batched kernel (SURVEY.md 8(f) f1); approx: hardware tanh in the "
                         "batch-1 gates (f4); appc: the paper's App. C approximations (f4; parity against "
                         "the oracle's App. C mode)")
    ap.add_argument("--samples", type=int, default=0, help="override samples per utterance (0 = workload's)")
    ap.add_argument("--streams", type=int, default=0,
                    help="override streams per GPU (0 = workload's; e.g. C2 with 8 streams = one cluster each)")
    ap.add_argument("--ref-samples", type=int, default=1600, help="samples per reference step")
    ap.add_argument("--cpu-samples", type=int, default=16000, help="oracle samples for cpu_baseline")
    ap.add_argument("--with-conditioner", action="store_true",
                    help="start each step from frame-rate features: the GPU QRNN conditioner (row f2) "
                         "runs inside the timed step before generation")
    ap.add_argument("--as-shard-of", type=int, default=1,
                    help="split workloads (C5): run rank 0's shard of a G-GPU job on this one GPU")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    wl = dict(WORKLOADS[args.workload])
    if args.samples:
        wl["n"] = args.samples
        wl["desc"] += f" [overridden: {args.samples} samples per utterance]"
    if args.streams:
        wl["streams"] = args.streams
        wl["desc"] += f" [overridden: {args.streams} streams]"
    if args.impl == "reference":
        return run_reference(args, wl)

    import torch
    ws, rank, local = dist_env()
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local if ws > 1 else 0)
    torch.cuda.set_device(dev)
    from paper_1702_07825_b200._lib import Conditioner, Model
    from paper_1702_07825_b200.shard import gather_codes, generate_sharded, shard_range

    cfg, n = wl["cfg"], wl["n"]
    if wl["split"] and args.as_shard_of > 1 and ws == 1:
        # one GPU runs exactly the block rank 0 of a G-GPU job would run (per-GPU rate at that G;
        # no collective on the path, so the G-GPU aggregate is G x this when ranks are alike)
        start, S = shard_range(wl["streams"], args.as_shard_of, 0)
    elif wl["split"]:
        start, S = shard_range(wl["streams"], ws, rank)
    else:
        S = wl["streams"]
        start = rank * S
    utts = list(range(start, start + S))
    w = synth.make_weights(cfg, 0)
    if S == 1:
        cond_np = synth.make_cond(cfg, synth.n_frames_for(n, HOP), utts[0])
        u_np = synth.make_uniforms(n, utts[0])
        d_cond = torch.from_numpy(cond_np)[None].to(dev)
        d_u = torch.from_numpy(u_np)[None].to(dev)
    else:
        d_cond, d_u = device_inputs(cfg, n, utts, dev)
    model = Model.from_config(cfg, device=dev.index).load(w).set_kernel(args.kernel).set_precision(args.precision)
    cond_net, d_feat = None, None
    if args.with_conditioner:  # features resident in HBM; cond is produced inside the step
        nf = synth.n_frames_for(n, HOP)
        cw = synth.make_conditioner_weights(synth.COND_FEATURES, synth.COND_HIDDEN, cfg.n_layers, cfg.residual, 0)
        cond_net = Conditioner(synth.COND_FEATURES, synth.COND_HIDDEN, cfg.n_layers, cfg.residual,
                               device=dev.index).load(cw)
        if S == 1:
            d_feat = torch.from_numpy(synth.make_features(nf, utt=utts[0]))[None].to(dev)
        else:
            d_feat = (torch.rand((S, nf, synth.COND_FEATURES), generator=torch.Generator(device=dev).manual_seed(7),
                                 device=dev) < 0.02).float()
        cond_net.run(d_feat, out=d_cond)
    stream = torch.cuda.current_stream(dev)
    out = torch.empty((S, n), dtype=torch.uint8, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2

    def barrier():
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize(dev)

    def step():
        if cond_net is not None:
            cond_net.run(d_feat, out=d_cond)
        model.generate(d_cond, d_u, HOP, out=out)

    n_utts = (S if args.as_shard_of > 1 else wl["streams"]) if wl["split"] else S * ws
    for i in range(args.warmup):
        if i == 0 and cond_net is None:
            # the first warm-up step through the sharder: this rank's contiguous block of the
            # n_utts utterances (PAPER.md:416 independent utterances; no collective)
            def resident(ids):
                assert list(ids) == utts, (ids[:3], utts[:3])
                return d_cond, d_u
            local, _, _ = generate_sharded(model, resident, n_utts, n, HOP, gather=False)
            out.copy_(local)
        else:
            step()
    barrier()
    info = model.info()
    floor = None
    if info["last_kernel_name"] == "cluster":
        from paper_1702_07825_b200._lib import measure_floor
        floor = measure_floor(dev.index)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(dev.index) as clk:
        barrier()
        for i in range(args.steps):
            flush.zero_()  # evict L2 between timed steps (untimed: outside the events)
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
        barrier()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    kernel_ms = float(np.mean(step_ms))
    model.sync()
    gpu_codes0 = out[0].cpu().numpy().copy()

    # end to end through the public host-buffer entry point (H2D + generate + D2H per step)
    e2e_step, h2d = None, int(d_cond.numel() * 4 + d_u.numel() * 4)
    if not args.no_e2e and h2d <= 16 * 2 ** 30 and cond_net is None:
        h_cond = d_cond.cpu().pin_memory()
        h_u = d_u.cpu().pin_memory()
        h_out = torch.empty((S, n), dtype=torch.uint8).pin_memory()
        model.generate_host(h_cond, h_u, HOP, out=h_out)
        barrier()
        e2e_ms = []
        for i in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            model.generate_host(h_cond, h_u, HOP, out=h_out)
            e2e_ms.append((time.perf_counter() - t0) * 1e3)
        e2e_step = float(np.mean(e2e_ms))
        assert np.array_equal(h_out[0].numpy(), gpu_codes0), "host-buffer path disagrees with device path"

    # batch 1: per-sample latency at 1,000-sample granularity -- the same
    # utterance through a streaming session in 1,000-sample chunks, CUDA events per chunk
    latency = None
    # (exact tiers only: approximate-tier sessions run on the stream kernel, not the one timed)
    if (S == 1 and cond_net is None and info["last_kernel_name"] in ("cluster", "stream") and n >= 2000
            and args.precision in ("fp32", "tf32")):
        sess = model.session(1)
        chunk = 1000
        cev = []
        for c0 in range(0, n, chunk):
            k = min(chunk, n - c0)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            sess.generate(d_cond, d_u[:, c0:c0 + k].contiguous(), HOP, out=out[:, c0:c0 + k])
            b.record(stream)
            cev.append((a, b, k))
        torch.cuda.synchronize(dev)
        per = np.array([a.elapsed_time(b) * 1e3 / k for a, b, k in cev])  # us per sample, per chunk
        assert np.array_equal(out[0].cpu().numpy(), gpu_codes0), "chunked session disagrees with one call"
        latency = {"us_per_sample_mean": float(per.mean()), "us_per_sample_p50": float(np.percentile(per, 50)),
                   "us_per_sample_p99": float(np.percentile(per, 99)), "chunks": len(per), "chunk_samples": chunk,
                   "first_chunk_ms": cev[0][0].elapsed_time(cev[0][1]),
                   "note": "streaming session (dvw_session_generate), 1,000-sample chunks incl. one launch each; "
                           "codes equal to the one-call run"}
        sess.close()

    # batch 1: teacher-forced logits of the same utterance on its own codes (dvw_logits, AUTO ->
    # the parallel-over-time kernel, tcgen05 at r = 64 / 128), outside the timed region
    tf_logits = None
    if S == 1 and cond_net is None:
        model.set_kernel("auto")
        codes_dev = torch.from_numpy(gpu_codes0)[None].to(dev)
        lg_buf = torch.empty((1, n, 256), dtype=torch.float32, device=dev)
        model.logits(d_cond, codes_dev, HOP, out=lg_buf)
        lev = []
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            model.logits(d_cond, codes_dev, HOP, out=lg_buf)
            b.record(stream)
            lev.append((a, b))
        torch.cuda.synchronize(dev)
        lms = float(np.median([a.elapsed_time(b) for a, b in lev]))
        linfo = model.info()
        tf_logits = {"ms_per_utterance": lms, "samples_per_s": n / (lms / 1e3), "kernel": linfo["last_kernel_name"],
                     "launches": int(linfo["last_launches"]),
                     "note": "dvw_logits on the generated codes (pre-softmax, all timesteps of a layer at once); "
                             "not part of the metric; its parity with the oracle is tested "
                             "(tests/test_gpu_parity.py, full C2 utterance)"}
        model.set_kernel(args.kernel)
        del lg_buf

    # max over ranks
    t_max, e_max = kernel_ms, (e2e_step if e2e_step is not None else -1.0)
    total_streams = S
    gather = None
    if ws > 1:
        # results to rank 0 after the timed work: the only collective (NCCL all_gather of uint8 codes)
        g0 = torch.cuda.Event(enable_timing=True)
        g1 = torch.cuda.Event(enable_timing=True)
        torch.distributed.barrier()
        g0.record(stream)
        full = gather_codes(out, n_utts)
        g1.record(stream)
        torch.cuda.synchronize(dev)
        gather = {"ms": g0.elapsed_time(g1), "bytes": int(n_utts * n), "utterances": n_utts,
                  "ok": (full is None) or (tuple(full.shape) == (n_utts, n) and bool(torch.equal(full[start:start + S],
                                                                                              out)))}
        import torch.distributed as dist
        t = torch.tensor([kernel_ms, e_max], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_max, e_max = float(t[0]), float(t[1])
        c = torch.tensor([S], device=dev)
        dist.all_reduce(c)
        total_streams = int(c[0])

    if rank == 0:
        total = n * total_streams
        value = total / (t_max / 1e3)
        flop_launch = 2.0 * macs_per_sample(cfg) * n * S
        achieved_tflops = flop_launch / (kernel_ms / 1e3) / 1e12
        kname = info["last_kernel_name"]
        fast = kname == "tc" and args.precision != "fp32"
        line_hbm = None
        if kname == "tc":
            peak, peak_src = tf32_peak_tflops()
            traffic = load_ncu_traffic(args.workload, n * S)
            if traffic is not None:  # the north_star's second batched-mode figure: HBM GB/s
                hpk, hsrc = hbm_peak_gbs()
                hgbs = traffic / (kernel_ms / 1e3) / 1e9
                line_hbm = {"achieved_gbs": hgbs, "peak_gbs": hpk, "frac": hgbs / hpk,
                            "note": f"ncu DRAM bytes per stream-sample x stream-samples / launch time, {hsrc}"}
            roof = {"bound": "tensor", "achieved": achieved_tflops, "peak": peak, "unit": "TFLOP/s",
                    "frac": achieved_tflops / peak, "traffic": traffic,
                    "note": "algorithmic FLOP (2 x MAC/sample x samples x streams) / launch time vs dense tf32 "
                            f"peak ({peak_src}); " + ("one tf32 pass (DVW_PRECISION_TF32); " if fast else
                            "the 3-pass split issues ~3.2x these FLOPs on the tensor pipe; ") +
                            "the step is phase-latency bound (DESIGN.md Batched kernel)"}
        elif kname == "cluster" and S > 1:
            # several streams interleaved per cluster (DESIGN.md §4.1 multi-stream variant): a throughput
            # kernel, bounded per cluster by its chain CTAs' issue slots; report the algorithmic FP32 rate
            # against the FFMA peak of the SMs the launch occupies at once (co-resident clusters x size)
            ghz = (clk.summary().get("sm_mhz") or 1965.0) / 1e3
            co = info["max_clusters_pipe"] if info["streams_per_cluster"] > 1 else info["max_clusters"]
            act = min(int(info["last_grid"]), int(co) * int(info["last_cluster"]))
            act_peak = act * 128 * 2 * ghz / 1e3
            roof = {"bound": "alu", "achieved": achieved_tflops, "peak": act_peak, "unit": "TFLOP/s",
                    "frac": achieved_tflops / act_peak, "active_sms": act,
                    "streams_per_cluster": int(info["streams_per_cluster"]),
                    "chip_fp32_peak_tflops": FP32_FMA_PEAK_TFLOPS,
                    "traffic": None,
                    "note": "multi-stream cluster kernel: algorithmic FLOP (2 x MAC/sample x samples x streams) "
                            "/ launch time vs the FP32 FFMA peak of the SMs it occupies at once (128 lanes x 2 x "
                            "SM clock each); per item the chain CTAs' serial layer work and their aux warps' "
                            "L2 weight streaming bound it (DESIGN.md §4.1)"}
        elif kname == "cluster" and floor is not None:
            # batch 1 is latency-bound: the roofline is the measured latency floor
            # of the critical path, l x layer + (chain CTAs + 2) x hop + 3 x head stage + sampler,
            # each piece microbenchmarked on this GPU now (dvw_measure_floor)
            nc = int(info["chain_ctas"])
            fc = (cfg.n_layers * floor["layer_cycles"] + (nc + 2) * floor["hop_cycles"]
                  + 3 * floor["head_stage_cycles"] + floor["sampler_cycles"])
            ghz = (clk.summary().get("sm_mhz") or floor["sm_ghz"] * 1e3) / 1e3
            floor_us = fc / ghz / 1e3
            us = kernel_ms * 1e3 / n
            peak = 1e6 / floor_us  # samples/s per stream at the floor
            roof = {"bound": "latency", "achieved": 1e6 / us, "peak": peak, "unit": "samples/s per stream",
                    "frac": floor_us / us, "floor_us": floor_us, "us_per_sample": us,
                    "traffic": load_ncu_traffic(args.workload, n * S),
                    "floor_parts_cycles": {"layer": floor["layer_cycles"], "hop": floor["hop_cycles"],
                                           "head_stage": floor["head_stage_cycles"],
                                           "sampler": floor["sampler_cycles"], "n_layers": cfg.n_layers,
                                           "hops": nc + 2, "head_stages": 3, "total": fc,
                                           "sm_ghz_probe": floor["sm_ghz"], "sm_ghz_used": ghz},
                    "alu": {"achieved_tflops": achieved_tflops, "chip_fp32_peak_tflops": FP32_FMA_PEAK_TFLOPS,
                            "frac": achieved_tflops / FP32_FMA_PEAK_TFLOPS},
                    "note": "frac = measured latency floor / measured us per sample (dvw_measure_floor: one "
                            "chain layer alone on an SM, one DSMEM hop, one head stage, one sampler draw; "
                            "DESIGN.md Roofline); alu = whole-chip FP32 context"}
            roof.update(load_active_sm_pipes(args.workload))
        else:
            roof = {"bound": "alu", "achieved": achieved_tflops, "peak": FP32_FMA_PEAK_TFLOPS,
                    "unit": "TFLOP/s", "frac": achieved_tflops / FP32_FMA_PEAK_TFLOPS,
                    "traffic": load_ncu_traffic(args.workload, n * S),
                    "note": "batch-1 is latency-bound: algorithmic FLOP (2 x MAC/sample x samples) / "
                            "launch time vs FP32 FFMA peak of the whole chip (DESIGN.md Roofline)"}
        line = {
            "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_max, "higher_is_better": True,
            "scaling": "strong" if wl["split"] else "weak",
            "vs_baseline": None,
            "dtype": ({"approx": "f32 (hardware tanh.approx gate)",
                       "appc": "f32 (App. C tanh/sigma/exp approximations)"}.get(args.precision, "f32") if kname != "tc"
                      else ("tf32 (1 tensor pass, inputs rounded to tf32)" if fast else "f32 (tf32 x3 tensor passes)")),
            "data": "synthetic",
            "config": {"workload": wl["desc"], "samples_per_step": n, "streams_per_gpu": S,
                       "streams_total": total_streams,
                       "parallelism": (f"{ws} GPU(s), independent utterances, no collective on the path"
                                       if args.as_shard_of <= 1 else
                                       f"1 GPU running rank 0's shard of a {args.as_shard_of}-GPU job "
                                       f"(the per-GPU rate at G = {args.as_shard_of}; not a multi-GPU run)"),
                       "kernel": kname, "grid": info["last_grid"], "cluster_ctas": info["last_cluster"],
                       "launches_per_step": info["last_launches"] + (5 if cond_net is not None else 0),
                       "conditioner": ("GPU QRNN (2 bidirectional fo-pooling layers, 227 features, 64 hidden) "
                                       "inside the timed step" if cond_net is not None else
                                       "synthetic conditioning (resident)"),
                       "l2": "flushed between timed steps (256 MiB write, untimed)"},
            "per_stream": {"samples_per_s": n / (kernel_ms / 1e3), "us_per_sample": kernel_ms * 1e3 / n,
                           "rtf_16khz": n / (kernel_ms / 1e3) / synth.AUDIO_HZ},
            "clocks": clk.summary(),
            "e2e": ({"value": total / (e_max / 1e3), "unit": "samples/s", "h2d_bytes_per_step": h2d,
                     "d2h_bytes_per_step": int(n * S)} if e_max > 0 else
                    {"value": None, "unit": "samples/s", "skipped": f"host inputs {h2d} B > 16 GiB, --no-e2e or --with-conditioner"}),
            "gpu_launches": (int(info["last_launches"]) + (5 if cond_net is not None else 0)) * args.steps,
            "roofline": roof,
        }
        if line_hbm is not None:
            line["hbm"] = line_hbm
        if gather is not None:
            line["gather_results"] = gather
        if latency is not None:
            line["latency"] = latency
        if tf_logits is not None:
            line["teacher_forced_logits"] = tf_logits
        if not args.no_cpu:
            cond0 = d_cond[0].cpu().numpy()
            u0 = d_u[0].cpu().numpy()
            k = min(n, 1600)
            model.set_kernel(kname)  # the teacher-forced check runs on the kernel that was timed
            tf = model.logits(d_cond[0:1].contiguous(), out[0:1, :k].contiguous(), HOP)[0].cpu().numpy()
            cpu, parity = cpu_baseline_and_parity(cfg, n, w, cond0, u0, gpu_codes0, args.cpu_samples, tf,
                                                  nonlin="appc" if args.precision == "appc" else "exact")
            cpu["cpu_model"] = cpu_model()
            cpu["host_threads"] = len(os.sched_getaffinity(0))
            if rank == 0 and args.workload in ("C1", "C2"):
                cpu["c1"] = cpu_c1_aggregate()
            line["cpu_baseline"] = cpu
            line["parity"] = parity
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
