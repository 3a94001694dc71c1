#!/usr/bin/env python
"""Benchmark of the sparse-causal chunk-attention hot path (BASELINE.json metric:
"chunk-attention TFLOP/s & ms/chunk (frac of bf16 peak) at 1/2/4/8 B200").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl tm|reference]
                    [--config wan512|wan720]

Workload (BASELINE.json configs[1]; configs[2] for N > 1): one WAN-2.1-14B-
shaped attention layer, H=40, d=128, 512x512 video -> 1024 tokens per latent
frame, reference c_0 = 1 latent frame (Lr=1024), chunk = 3 latent frames
(Lc=3072), chunk index t >= 2 so the attend set is {c_0, c_{t-1}, c_t}
(Lk = 7168; Eq 7).  FLOP per call = 4*Lc*Lk*d*H = 450.97 GFLOP
(algorithmic: allowed keys only, QK^T + PV).

One STEP = one pass of the hot path over one chunk at one (layer, step):
  a2/a3 (Ulysses exchange for N>1 / K,V append into cache slot t&1)
  a4    mask -> segment schedule
  a5    tcgen05 attention over {c_0, c_{t-1}, c_t}
  a6    (N>1) head -> seq exchange of O
  a7    flow-matching Euler update of the chunk latent (16 x 3 x 64 x 64)
The reference K/V (a1) is written once per stream per (layer, step) in setup,
as the paper caches it.  Steps rotate over 8 layers' caches and 4
input sets (~210 MB touched per step, > 126 MB L2), so every step reads its
operands from HBM ("inputs larger than L2").

N > 1: heads are sharded across ranks (H/N per rank), each rank passes its
sequence shard [Lc/N][H][d]; the library runs the Ulysses all-to-all (NCCL)
in and out.  Total work is fixed -> "scaling": "strong".

--impl reference: the fp64 CPU oracle (oracle/) timed on the host cores on a
bounded row sample of the same workload (this tier has no reference code).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "chunk-attention TFLOP/s & ms/chunk (frac of bf16 peak) at 1/2/4/8 B200"
CONFIGS = {
    "wan512": dict(H=40, d=128, Lr=1024, Lc=3072, latent=16 * 3 * 64 * 64,
                   workload="WAN-2.1-14B-shaped single layer, 512x512 (1024 tok/frame), "
                            "chunk t>=2 = 3 latent frames + cached reference frame + previous chunk"),
    "wan512c7": dict(H=40, d=128, Lr=1024, Lc=7168, latent=16 * 7 * 64 * 64,
                     workload="Table 1 variant (P:249-258): WAN-2.1-14B-shaped layer, 512x512, "
                              "chunk = 7 latent frames + cached reference frame + previous chunk"),
    "wan720": dict(H=40, d=128, Lr=2025, Lc=6075, latent=16 * 3 * 90 * 90,
                   workload="WAN-2.1-14B-shaped single layer, 720x720 (2025 tok/frame), "
                            "chunk t>=2 = 3 latent frames + cached reference frame + previous chunk"),
}
FALLBACK_PEAK_TFLOPS = 1590.0     # /opt/skills/guides/B200_PROFILING.md fallback


def flop_per_call(c, t=2):
    Lk = c["Lr"] + (2 if t >= 2 else 1) * c["Lc"]
    return 4.0 * c["Lc"] * Lk * c["d"] * c["H"]


def algo_bytes(c, t=2):
    """HBM bytes one launch must move (bf16): reads Q, K/V of the reference,
    previous and current chunks; writes O and (a3, fused) the current K/V into
    the cache slot."""
    row = c["H"] * c["d"] * 2
    reads = c["Lc"] * row + 2 * c["Lr"] * row + 2 * (2 if t >= 2 else 1) * c["Lc"] * row
    writes = c["Lc"] * row + 2 * c["Lc"] * row
    return float(reads + writes)


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            j = json.load(f)
        return float(j["bf16_tflops"]), float(j.get("bf16_tflops_sustained", 0)), "measured"
    except Exception:
        return FALLBACK_PEAK_TFLOPS, None, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons, polled every 20 ms around the timed
    regions; summary(window) keeps the samples taken inside a wall-clock window."""

    FIELDS = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    REASONS = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, device_index):
        self.dev = device_index
        self.proc = None
        self.tmp = None
        self.rows = []

    def start(self, settle=1.5):
        """Start polling; wait `settle` s so nvidia-smi's NVML start-up (which can
        stall CUDA launches from this process) is over before timing starts."""
        try:
            self.tmp = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.dev}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=self.tmp, stderr=subprocess.DEVNULL)
            time.sleep(settle)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return
        time.sleep(0.1)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.tmp.flush()
        self.tmp.seek(0)
        self.rows = [r.split(",") for r in self.tmp.read().strip().splitlines() if r.strip()]
        os.unlink(self.tmp.name)

    @staticmethod
    def _ts(r):
        import datetime
        try:
            return datetime.datetime.strptime(r[0].strip(), "%Y/%m/%d %H:%M:%S.%f").timestamp()
        except Exception:
            return None

    def summary(self, window=None):
        rows = self.rows
        inside = False
        if window is not None:
            sel = [r for r in rows if self._ts(r) is not None and window[0] <= self._ts(r) <= window[1]]
            if sel:
                rows, inside = sel, True
        sm, smax, reasons = [], 0.0, set()
        for r in rows:
            try:
                sm.append(float(r[1]))
                smax = max(smax, float(r[2]))
                for nm, val in zip(self.REASONS, r[5:9]):
                    if "Active" in val and "Not" not in val:
                        reasons.add(nm)
            except Exception:
                continue
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm), "in_timed_window": inside}


class NvmlSampler:
    """In-process NVML polling (~1 ms) of the SM clock and clock-event reasons
    from a thread, so that even a ~13 ms timed region gets samples (the
    nvidia-smi poller's 20 ms period can miss it)."""

    BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
            "hw_thermal_slowdown": 0x40}

    def __init__(self, device_index):
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.smax = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
            self.ok = True
        except Exception:
            pass
        self.samples = []
        self.thread = None

    def _reasons(self):
        nv = self.nv
        f = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        return int(f(self.h))

    def start(self):
        import threading
        if not self.ok:
            return
        self.samples = []
        self.stop_flag = False

        def loop():
            while not self.stop_flag:
                try:
                    self.samples.append((float(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)),
                                         self._reasons()))
                except Exception:
                    pass
                time.sleep(0.001)

        self.thread = threading.Thread(target=loop, daemon=True)
        self.thread.start()

    def stop(self):
        if self.thread:
            self.stop_flag = True
            self.thread.join(timeout=2)
            self.thread = None

    def summary(self):
        if not self.samples:
            return None
        reasons = sorted(nm for nm, bit in self.BITS.items() if any(r & bit for _, r in self.samples))
        return {"sm_mhz": statistics.median(c for c, _ in self.samples), "sm_max_mhz": self.smax,
                "reasons": reasons, "samples": len(self.samples), "in_timed_window": True,
                "source": "NVML, ~1 ms polling thread"}


# ----------------------------------------------------------------------------- reference arm

_ORACLE_INPUTS = {}


def _oracle_inputs(c, seed):
    """Seeded synthetic inputs of one t>=2 call (generated once, reused)."""
    key = (c["H"], c["d"], c["Lr"], c["Lc"], seed)
    if key not in _ORACLE_INPUTS:
        from synthetic import inputs as syn
        si = syn.StreamInputs(c["H"], c["d"], c["Lr"], c["Lc"], "bf16", "D0", seed)
        _, kr, vr = si.chunk(0, 0, 0)
        _, kp, vp = si.chunk(0, 0, 1)
        q, kc, vc = si.chunk(0, 0, 2)
        _ORACLE_INPUTS[key] = [t.f64 for t in (q, kr, vr, kp, vp, kc, vc)]
    return _ORACLE_INPUTS[key]


def run_oracle_sample(c, rows, seed, offset=0):
    """Oracle (fp64 C, OpenMP) on `rows` query rows x all heads of one t>=2
    call; returns (seconds, flop, threads)."""
    import numpy as np
    import oracle
    q, kr, vr, kp, vp, kc, vc = _oracle_inputs(c, seed)
    r = (np.linspace(0, c["Lc"] - 1, rows).astype(np.int64) + offset) % c["Lc"]
    t0 = time.perf_counter()
    oracle.stream_attention(q, kr, vr, kp, vp, kc, vc, rows=r)
    dt = time.perf_counter() - t0
    Lk = c["Lr"] + 2 * c["Lc"]
    return dt, 4.0 * rows * Lk * c["d"] * c["H"], oracle.num_threads()


def reference_arm(args, c):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    rows = args.oracle_rows
    times, flops = [], 0.0
    threads = 0
    for s in range(args.warmup):
        run_oracle_sample(c, max(8, rows // 8), 7, offset=s)
    for s in range(args.steps):
        dt, fl, threads = run_oracle_sample(c, rows, 7, offset=1 + s)
        times.append(dt)
        flops = fl
    total = sum(times)
    value = flops * args.steps / total / 1e12
    sample = (f"{rows} query rows x {c['H']} heads of one t>=2 call (Lk={c['Lr'] + 2 * c['Lc']}), "
              f"per step; fp64 two-pass softmax over the literal concatenation")
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s",
           "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": c["workload"], "heads": c["H"], "head_dim": c["d"],
                      "ref_tokens": c["Lr"], "chunk_tokens": c["Lc"], "chunk_index": 2},
           "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": threads, "kind": "oracle",
                            "sample": sample, "cpu_model": cpu_model(), "nproc": os.cpu_count()},
           "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


# ----------------------------------------------------------------------------- Sec 8(f) rows

def _time_ms(torch, fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ev = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        ev.append((a, b))
    torch.cuda.synchronize()
    return statistics.median(x.elapsed_time(y) for x, y in ev)


def _loop_ms(torch, fn, reps, warm=5):
    """ms per call of `reps` calls back to back between one event pair."""
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def _graph_ms(torch, fn, reps, R=5):
    """ms per call of `reps` calls captured in one CUDA graph, replayed R times
    (median): the GPU time without host work between launches."""
    fn()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(R):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / reps)
    del g
    return statistics.median(ts)


def measured_hbm():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except Exception:
        return 6650.0                  # /opt/skills/guides/B200_PROFILING.md fallback


def measure_extras(tm, c, torch, stream):
    """SURVEY Sec 8(f) rows at WAN shapes, random data: f1 full 21-frame window,
    f2 fused sampler step (HBM roofline), f4 audio cross-attention."""
    H, d = c["H"], c["d"]
    bf = torch.bfloat16
    g = torch.Generator(device="cuda").manual_seed(2506030990 + 77)
    out = {}
    # f1: 7 chunks x 3 latent frames of 1024 tokens
    lens = [3 * 1024] * 7
    L = sum(lens)
    q, k, v = (torch.randn(L, H, d, device="cuda", dtype=bf, generator=g) for _ in range(3))
    o = torch.empty_like(q)
    ca = tm.ChunkAttention(H, d, 16, 16, 1, 1)
    ms = _time_ms(torch, lambda: ca.window(q, k, v, o, lens))
    Lc = lens[0]
    fl = 4.0 * d * H * Lc * Lc * (1 + 2 + 3 * 5)
    out["f1_window"] = {"workload": "21-latent-frame window, 7 chunks x 3072 tokens, 40 heads",
                        "ms": ms, "tflops": fl / (ms * 1e-3) / 1e12, "gflop": fl / 1e9}
    del q, k, v, o
    # f2: one sampler step over 64 chunks' latents (16 ch x 3 x 64 x 64 each).
    # HBM-bound kernels: 4 operand sets rotated (x, v, x_bf16: 100 MB per set,
    # 400 MB in all > the 126 MB L2), so every call streams from HBM; K calls
    # back to back between one event pair.
    n = 64 * 16 * 3 * 64 * 64
    NS = 4
    xs = [torch.randn(n, device="cuda", generator=g) for _ in range(NS)]
    vs = [torch.randn(n, device="cuda", generator=g).to(bf) for _ in range(NS)]
    xbs = [torch.empty(n, device="cuda", dtype=bf) for _ in range(NS)]
    es = [torch.randn(n, device="cuda", generator=g) for _ in range(NS)]
    cnt = [0]

    def sampler():
        i = cnt[0] % NS
        cnt[0] += 1
        tm.tm_flow_sampler_step(ca.ctx, xs[i], vs[i], tm.TM_BF16, n, 0.0, 0.5, seed=1,
                                x_bf16_out=xbs[i])

    def sampler_eps():
        i = cnt[0] % NS
        cnt[0] += 1
        tm.tm_flow_sampler_step(ca.ctx, xs[i], vs[i], tm.TM_BF16, n, 0.0, 0.5, eps=es[i],
                                x_bf16_out=xbs[i])

    def euler():
        i = cnt[0] % NS
        cnt[0] += 1
        tm.tm_flow_euler_step(ca.ctx, xs[i], vs[i], tm.TM_BF16, n, 0.5)

    hbm = measured_hbm()
    ms = _loop_ms(torch, sampler, 40)
    byts = n * (4 + 4 + 2 + 2)        # x read + write, v bf16, bf16 copy; noise in-kernel
    out["f2_sampler"] = {"workload": f"{n} elements (64 chunks of 16x3x64x64), in-kernel Philox",
                         "ms": ms, "gbs": byts / (ms * 1e-3) / 1e9, "bytes": byts,
                         "frac_of_hbm": byts / (ms * 1e-3) / 1e9 / hbm, "bound": "hbm",
                         "timing": f"40 calls back to back, {NS} operand sets rotated (> L2)",
                         "note": "in-kernel Philox4x32-10 + Box-Muller with an accurate logf: "
                                 "~50 instructions per element, issue-bound (ncu: issue slots "
                                 "~70% busy); the caller-noise form below is the HBM-bound one"}
    ms = _loop_ms(torch, sampler_eps, 40)
    byts = n * (4 + 4 + 2 + 4 + 2)    # x read + write, v bf16, eps fp32, bf16 copy
    out["f2_sampler_given_noise"] = {
        "workload": f"{n} elements, noise eps passed by the caller (fp32)", "ms": ms,
        "gbs": byts / (ms * 1e-3) / 1e9, "bytes": byts,
        "frac_of_hbm": byts / (ms * 1e-3) / 1e9 / hbm, "bound": "hbm",
        "timing": f"40 calls back to back, {NS} operand sets rotated (> L2)"}
    # a7 at the same size (report GB/s at n = 12.6 M)
    ms = _loop_ms(torch, euler, 40)
    byts = n * (4 + 4 + 2)
    out["a7_euler_12.6M"] = {"ms": ms, "gbs": byts / (ms * 1e-3) / 1e9, "bytes": byts,
                             "frac_of_hbm": byts / (ms * 1e-3) / 1e9 / hbm, "bound": "hbm",
                             "timing": f"40 calls back to back, {NS} operand sets rotated (> L2)"}
    del xs, vs, xbs, es
    # f4: a chunk of 3 frames, 16x16 face region, 32 audio tokens per frame
    frames, T, A = 3, 1024, 32
    qa = torch.randn(frames, T, H, d, device="cuda", dtype=bf, generator=g)
    ka = torch.randn(frames, A, H, d, device="cuda", dtype=bf, generator=g)
    va = torch.randn(frames, A, H, d, device="cuda", dtype=bf, generator=g)
    oa = torch.empty_like(qa)
    face = torch.tensor([r * 32 + cc for r in range(8, 24) for cc in range(8, 24)], dtype=torch.int32,
                        device="cuda")
    ms = _loop_ms(torch, lambda: ca.audio(qa, ka, va, oa, face, stream=stream), 40)
    ms_g = _graph_ms(torch, lambda: ca.audio(qa, ka, va, oa, face), 40)
    fl = 4.0 * frames * face.numel() * 5 * A * d * H
    byts = (frames * T * H * d * 2) * 2 + 2 * frames * A * H * d * 2
    ms_best = min(ms, ms_g)
    out["f4_audio"] = {"workload": "3 latent frames x 1024 tokens, 256 face tokens, window 5 x 32 "
                                   "audio tokens, 40 heads", "ms": ms_best, "ms_graph": ms_g,
                       "ms_eager": ms, "launches_per_call": ca.launches,
                       "timing": "ms = the lower of two event-pair timings of 40 calls, each an upper "
                                 "bound of the GPU time: ms_eager (calls from Python, back to back; "
                                 "host-bound when the ~20 us of binding + launch work per call "
                                 "exceeds the GPU time) and ms_graph (the same calls captured in one "
                                 "CUDA graph, median of 5 replays)",
                       "tflops": fl / (ms_best * 1e-3) / 1e12, "gbs_io": byts / (ms_best * 1e-3) / 1e9}
    ca.close()
    return out


def stored_traffic(config, P):
    """DRAM bytes per launch of the dominant kernel from the committed ncu
    --set full capture (profiles/ncu_fmha_traffic.json): ncu cannot run inside
    the bench, so `traffic` is the STORED figure of that capture, labelled."""
    prof = os.path.join(ROOT, "profiles", "ncu_fmha_traffic.json")
    try:
        with open(prof) as f:
            pj = json.load(f)
        if pj.get("config") == config and pj.get("n_gpus") == P:
            return pj.get("dram_bytes_per_launch"), \
                f"stored: profiles/ncu_fmha_traffic.json ({pj.get('source', 'ncu --set full')})"
    except Exception:
        pass
    return None, "no stored ncu capture for this config"


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def cpu_baseline(c, rows):
    """The oracle as it stands, on all host cores and on one core (SURVEY
    Sec 8(d) oracle timing), on bounded row samples of one t>=2 call."""
    import oracle
    dt, sfl, th = run_oracle_sample(c, rows, 7)
    one_rows = max(8, rows // 16)
    oracle.set_num_threads(1)
    try:
        dt1, sfl1, _ = run_oracle_sample(c, one_rows, 7, offset=3)
    finally:
        oracle.set_num_threads(th)
    Lk = c["Lr"] + 2 * c["Lc"]
    return {"value": sfl / dt / 1e12, "unit": "TFLOP/s", "cores": th, "kind": "oracle",
            "sample": f"{rows} query rows x {c['H']} heads of one t>=2 call (Lk={Lk}); {dt:.1f} s",
            "cpu_model": cpu_model(), "nproc": os.cpu_count(),
            "one_core": {"value": sfl1 / dt1 / 1e12, "unit": "TFLOP/s", "cores": 1,
                         "sample": f"{one_rows} query rows x {c['H']} heads; {dt1:.1f} s"},
            "extrapolated_full_call_s": {"all_cores": dt * c["Lc"] / rows,
                                         "one_core": dt1 * c["Lc"] / one_rows}}


def attention_loop(tm, torch, H, d, Lr, Lc, K, stream, zero_copy=False, NL=8, NB=4, sched_heads=0,
                   R=3, idle=0.0):
    """ms per chunk-attention call (t >= 2) of a fresh H-head context: K calls
    back to back between one event pair (median of R such loops), operands
    rotated over NL layer caches and NB input sets (larger than L2); fused c_t
    append unless zero_copy."""
    bf = torch.bfloat16
    g = torch.Generator(device="cuda").manual_seed(2506030990 + 55 + H)
    ca = tm.ChunkAttention(H, d, Lr, Lc, NL, 1, sched_heads=sched_heads)
    sets = [[torch.randn(Lc, H, d, device="cuda", dtype=bf, generator=g) for _ in range(3)]
            for _ in range(NB)]
    o = torch.empty(Lc, H, d, device="cuda", dtype=bf)
    kr = torch.randn(Lr, H, d, device="cuda", dtype=bf, generator=g)
    for layer in range(NL):
        ca.put_reference(layer, 0, kr, kr)
    chunk = [0] * NL

    def call(i):
        layer = i % NL
        chunk[layer] += 1
        q, k, v = sets[i % NB]
        if zero_copy and chunk[layer] >= 2:
            kp, vp = ca.slot_ptr(layer, 0, chunk[layer])
            # the slot holds c_{t-2}'s random K/V: realistic data, no copy
            k, v = kp, vp
        ca.attend(layer, 0, chunk[layer], q, k, v, o, stream)

    for i in range(3 * NL):
        call(i)
    torch.cuda.synchronize()
    ts = []
    for _ in range(R):
        if idle > 0:
            time.sleep(idle)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for i in range(K):
            call(i)
        b.record(stream)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / K)
    ca.close()
    del sets
    return statistics.median(ts)


def measure_other_configs(tm, torch, main, K, stream):
    """Driver-run lines for the other single-GPU configs of BASELINE.json
    (720^2, configs[4]) and the Table-1 chunk-7 shape: the
    attention-only loop of each (fused append, t >= 2)."""
    peak = measured_peaks()[0]
    out = {}
    for name in ("wan720", "wan512c7"):
        if name == main:
            continue
        cc = CONFIGS[name]
        # as long as the main timed region (~13 ms: a burst, not power-capped),
        # each of R = 3 loops after a 0.5 s idle
        Kc = max(3, int(round(K * flop_per_call(CONFIGS[main]) / flop_per_call(cc))))
        ms = attention_loop(tm, torch, cc["H"], cc["d"], cc["Lr"], cc["Lc"], Kc, stream, idle=0.5)
        fl = flop_per_call(cc)
        out[name] = {"workload": cc["workload"], "keys_attended": cc["Lr"] + 2 * cc["Lc"],
                     "ms_per_call": ms, "tflops": fl / (ms * 1e-3) / 1e12,
                     "frac_of_bf16_peak": fl / (ms * 1e-3) / 1e12 / peak,
                     "gflop_per_call": fl / 1e9,
                     "timing": f"{Kc} calls (fused append; the main region's FLOP) between one "
                               "event pair, median of 3 loops each after a 0.5 s idle"}
        torch.cuda.empty_cache()
    return out


# Peer-copy bandwidth per direction per GPU measured on this pool
# (/opt/skills/guides/B200_PROFILING.md), for the modelled exposed Q push.
NVLINK_PEER_GBS = 770.0


def measure_shards(tm, torch, c, K, stream, t1_ms):
    """One rank's share of the WAN-512 call at P = 2, 4, 8 (H/P heads) on one
    GPU -- the per-rank kernel of the Ulysses head sharding -- with
    the fused append (as the P > 1 call runs it) and zero-copy, and the scaling
    MODEL E(P) = t(1) / (P t(P)), t(P) = shard kernel + exposed Q push (remote
    share of this rank's Q shard at the measured 770 GB/s peer copy) + 1 us
    done barrier.  A model from one-GPU numbers, not a multi-GPU measurement.
    t(1) is re-measured with each shard (same loop, both after a 0.5 s idle:
    sustained loops run power-capped and a small-H loop right after a 40-head
    loop reads up to 20 % slow while the clocks recover, so t(1) and t(P) are
    only comparable when taken the same way; tools/dbg/shard_vs_bench.py)."""
    H, d, Lr, Lc = c["H"], c["d"], c["Lr"], c["Lc"]
    out = {"model": "t(P) = shard kernel (fused append) + exposed Q push at "
                    f"{NVLINK_PEER_GBS:.0f} GB/s + 1 us; E(P) = t(1) / (P t(P)); "
                    "t(1) = the 40-head loop timed with each shard, both after a 0.5 s idle",
           "t1_ms_live": t1_ms}
    for P in (2, 4, 8):
        Hs = H // P
        time.sleep(0.5)
        ms = attention_loop(tm, torch, Hs, d, Lr, Lc, K, stream)
        ms_zc = attention_loop(tm, torch, Hs, d, Lr, Lc, K, stream, zero_copy=True)
        time.sleep(0.5)
        t1 = attention_loop(tm, torch, H, d, Lr, Lc, K, stream)
        Ls = -(-Lc // P)
        q_push_us = Ls * H * d * 2 * (P - 1) / P / (NVLINK_PEER_GBS * 1e3)
        t = ms + (q_push_us + 1.0) * 1e-3
        fl = flop_per_call(c) / P
        out[f"h{Hs}"] = {"P": P, "heads": Hs, "t1_ms": t1, "ms_fused_append": ms,
                         "ms_zero_copy": ms_zc,
                         "tflops_fused_append": fl / (ms * 1e-3) / 1e12,
                         "tflops_zero_copy": fl / (ms_zc * 1e-3) / 1e12,
                         "q_push_us_model": q_push_us, "t_model_ms": t,
                         "E_model": t1 / (P * t), "E_kernel_only": t1 / (P * ms)}
    # P-invariant schedule (tm_config.sched_heads = H/8: every 5 heads scheduled
    # as a block of their own, bitwise equal outputs for P = 1, 2, 4, 8): its
    # cost at P = 1 against the default schedule, the same loop back to back.
    time.sleep(0.5)
    base = attention_loop(tm, torch, H, d, Lr, Lc, K, stream)
    inv = attention_loop(tm, torch, H, d, Lr, Lc, K, stream, sched_heads=H // 8)
    out["p_invariant_p1"] = {"sched_heads": H // 8, "ms_default": base, "ms_p_invariant": inv,
                             "cost_frac": inv / base - 1.0}
    return out


# ----------------------------------------------------------------------------- tm arm

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=8)
    ap.add_argument("--impl", default="tm", choices=["tm", "reference"])
    ap.add_argument("--config", default="wan512", choices=sorted(CONFIGS))
    ap.add_argument("--layers", type=int, default=8, help="layer caches rotated over")
    ap.add_argument("--oracle-rows", type=int, default=256)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the SURVEY Sec 8(f) rows (f1 window, f2 sampler, f4 audio)")
    ap.add_argument("--transport", default=None, choices=["peer", "nccl"],
                    help="Ulysses exchange for N>1 (default peer: fused NVLink peer-memory "
                         "push/scatter; nccl: pack + ncclAlltoAll + unpack).  At N=1 the "
                         "default is the direct path; --transport peer runs a 1-rank group.")
    ap.add_argument("--stream-chunks", type=int, default=64,
                    help="BJ.configs[3] streaming measurement over this many chunks (0: off)")
    args = ap.parse_args()
    # Watchdog: a rank stuck in a collective (a hung exchange is the realistic
    # multi-GPU failure) dumps its stacks and exits instead of holding the box.
    import faulthandler
    faulthandler.dump_traceback_later(int(os.environ.get("TM_BENCH_WATCHDOG_S", "1800")), exit=True)
    if args.warmup < 3:
        args.warmup = 3
    c = CONFIGS[args.config]
    if args.impl == "reference":
        reference_arm(args, c)
        return

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # Test hook (not a benchmark mode): TM_BENCH_ONE_DEVICE=1 puts every rank on
    # cuda:0 with a gloo process group, so the N>1 flow (peer windows over CUDA
    # IPC, barriers, max over ranks) can be exercised on a one-GPU box; the
    # time-sliced numbers it prints are meaningless.
    one_dev = os.environ.get("TM_BENCH_ONE_DEVICE") == "1"
    if one_dev:
        local = 0
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    if world > 1:
        if one_dev:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2506_03099_b200 import tm

    H, d, Lr, Lc = c["H"], c["d"], c["Lr"], c["Lc"]
    P = world
    Lc_s, Lr_s = -(-Lc // P), -(-Lr // P)
    NL = args.layers
    transport = args.transport or ("peer" if P > 1 else "nccl")
    if transport == "peer" and P > 1 and not one_dev:
        # the peer windows need NVLink/PCIe peer access between every pair of GPUs
        ok = all(torch.cuda.can_device_access_peer(local, j) for j in range(P) if j != local)
        flag = torch.tensor([1 if ok else 0], device="cuda", dtype=torch.int32)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if int(flag.item()) == 0:
            if rank == 0:
                print("bench: no peer access between all GPUs; using the NCCL transport",
                      file=sys.stderr)
            transport = "nccl"
    tcode = tm.TM_TRANSPORT_PEER if transport == "peer" else tm.TM_TRANSPORT_NCCL
    nccl_id = None
    if P > 1 and transport == "nccl":
        obj = [tm.tm_get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]

    def make_ctx(layers, steps):
        cx = tm.ChunkAttention(H, d, Lr, Lc, num_layers=layers, num_steps=steps, world_size=P,
                               rank=rank, device=local, nccl_id=nccl_id, transport=tcode)
        if transport == "peer" and P > 1:
            cx.connect_dist()          # CUDA IPC handles of the windows, all-gathered
        return cx

    ca = make_ctx(NL, 1)
    stream = torch.cuda.current_stream()
    g = torch.Generator(device="cuda").manual_seed(2506030990 + 1000 + rank)
    bf = torch.bfloat16
    NB = 4
    sets = [[torch.randn(Lc_s, H, d, device="cuda", dtype=bf, generator=g) for _ in range(3)]
            for _ in range(NB)]
    outs = [torch.empty(Lc_s, H, d, device="cuda", dtype=bf) for _ in range(NB)]
    if transport == "peer" and P > 1:
        # zero-copy output: the ranks' epilogues write straight into this rank's
        # O window, the receive phase only waits (tm_peer_output_ptr)
        outs = [ca.output_window()[0]] * NB
    xlat = torch.randn(c["latent"], device="cuda", generator=g)
    vlat = torch.randn(c["latent"], device="cuda", generator=g).to(bf)
    kref = torch.randn(Lr_s, H, d, device="cuda", dtype=bf, generator=g)
    vref = torch.randn(Lr_s, H, d, device="cuda", dtype=bf, generator=g)
    for layer in range(NL):                                    # a1, once per stream
        ca.put_reference(layer, 0, kref, vref, stream)
    chunk = [0] * NL
    launches = [0]

    def step(i, zero_copy=False, ev=None):
        layer = i % NL
        chunk[layer] += 1
        q, k, v = sets[i % NB]
        o = outs[i % NB]
        if zero_copy:
            k, v = ca.slot_ptr(layer, 0, chunk[layer])
        if ev is not None:
            ev[0].record(stream)
        ca.attend(layer, 0, chunk[layer], q, k, v, o, stream)
        if ev is not None:
            ev[1].record(stream)
        n = ca.launches
        ca.euler(xlat, vlat, tm.TM_BF16, 0.5, stream)
        launches[0] += n + ca.launches

    for i in range(NL):                                        # chunk 1 of every layer
        step(i)
    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()

    def barrier():
        if P > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if P == 1:
            return x
        t = torch.tensor([x], device="cpu" if one_dev else "cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---------------------------------------------------------------- main timed region
    clocks = ClockSampler(local)
    clocks.start()
    nvml = NvmlSampler(local)
    launches[0] = 0
    barrier()
    w0 = time.time()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    nvml.start()
    e0.record(stream)
    for i in range(args.steps):
        step(i)
    e1.record(stream)
    barrier()
    nvml.stop()
    w1 = time.time()
    ms_total = max_over_ranks(e0.elapsed_time(e1))
    gpu_launches = launches[0]

    # ---------------------------------------------------------------- dominant kernel, live
    # roofline.achieved: the same attention calls as the step (fused c_t append,
    # same input rotation) back to back, WITHOUT the Euler update, between ONE
    # event pair on the launching stream -- so the launches overlap exactly as
    # in the step (PDL) and the per-launch time cannot exceed ms_per_step.
    barrier()
    la0, la1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    la0.record(stream)
    for i in range(args.steps):
        layer = i % NL
        chunk[layer] += 1
        q, k, v = sets[i % NB]
        ca.attend(layer, 0, chunk[layer], q, k, v, outs[i % NB], stream)
    la1.record(stream)
    barrier()
    live_ms = max_over_ranks(la0.elapsed_time(la1) / args.steps)

    # ---------------------------------------------------------------- attention kernel alone
    # P = 1: K/V pre-placed in the cache slot (zero-copy append) so each call is
    # one attention-kernel launch.  P > 1: the whole call (peer: the fused
    # push + attention + scatter kernel and the receive kernel; nccl: pack,
    # all-to-all, unpack, attention, pack, all-to-all, unpack).  Per-call CUDA
    # events on the launching stream.
    kev = []
    zc = P == 1 and transport == "nccl"

    def kv_for(i, layer):
        if zc:
            return ca.slot_ptr(layer, 0, chunk[layer])
        return sets[i % NB][1], sets[i % NB][2]

    barrier()
    for i in range(3):          # fill the launch queue so no event pair spans a host gap
        layer = i % NL
        chunk[layer] += 1
        kp, vp = kv_for(i, layer)
        ca.attend(layer, 0, chunk[layer], sets[i % NB][0], kp, vp, outs[i % NB], stream)
    w2 = time.time()
    for i in range(args.steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        layer = i % NL
        chunk[layer] += 1
        q = sets[i % NB][0]
        kp, vp = kv_for(i, layer)
        a.record(stream)
        ca.attend(layer, 0, chunk[layer], q, kp, vp, outs[i % NB], stream)
        b.record(stream)
        kev.append((a, b))
    barrier()
    w3 = time.time()
    if P > 1 or transport == "peer":
        ca.check()      # peer: a device-side wait timed out; nccl: the communicator's async error
    clocks.stop()
    clk = nvml.summary() or clocks.summary(window=(w0, w1))
    kclk = clocks.summary(window=(w2, w3))
    k_list = [a.elapsed_time(b) for a, b in kev]
    k_ms = max_over_ranks(statistics.mean(k_list))
    k_med = max_over_ranks(statistics.median(k_list))

    # ---------------------------------------------------------------- chunk t = 1
    # The first chunk of a stream attends {c_0, c_1} only (Lk = Lr + Lc): a new
    # stream on the same context (tm_stream_reset), every layer's chunk 1 timed.
    ca.reset()
    for layer in range(NL):
        ca.put_reference(layer, 0, kref, vref, stream)
    ev1 = []
    barrier()
    for layer in range(NL):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        q, k, v = sets[layer % NB]
        a.record(stream)
        ca.attend(layer, 0, 1, q, k, v, outs[layer % NB], stream)
        b.record(stream)
        ev1.append((a, b))
    barrier()
    t1_ms = max_over_ranks(statistics.median(a.elapsed_time(b) for a, b in ev1))
    chunk[:] = [1] * NL        # the reset stream is at chunk 1 on every layer

    # ---------------------------------------------------------------- end to end, host buffers
    e2e = None
    if not args.no_e2e:
        # Host buffers through the public API, copies inside the timed region,
        # double-buffered: H2D of step i+1 (copy stream) and D2H of step i-1
        # overlap the kernels of step i (compute stream).
        hq = [t.cpu().pin_memory() for t in sets[0]]
        hx = xlat.cpu().pin_memory()
        hv = vlat.cpu().pin_memory()
        ho = [torch.empty(Lc_s, H, d, dtype=bf).pin_memory() for _ in range(2)]
        hxo = [torch.empty_like(hx).pin_memory() for _ in range(2)]
        dq = [[torch.empty_like(t) for t in sets[0]] for _ in range(2)]
        dx = [torch.empty_like(xlat) for _ in range(2)]
        dv = [torch.empty_like(vlat) for _ in range(2)]
        do = [torch.empty(Lc_s, H, d, device="cuda", dtype=bf) for _ in range(2)]
        h2d = sum(t.numel() * t.element_size() for t in hq) + hx.numel() * 4 + hv.numel() * 2
        d2h = ho[0].numel() * 2 + hx.numel() * 4
        s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
        ke = max(3, min(args.steps, 24))     # steps; the pipeline fill is amortised over them
        ev = lambda: torch.cuda.Event(enable_timing=False)
        in_ready = [None, None]
        out_done = [None, None]
        barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s_in)
        stream.wait_stream(s_in)
        s_out.wait_stream(s_in)
        for i in range(ke):
            j = i % 2
            with torch.cuda.stream(s_in):
                if out_done[j] is not None:
                    s_in.wait_event(out_done[j])
                for dst, src in zip(dq[j], hq):
                    dst.copy_(src, non_blocking=True)
                dx[j].copy_(hx, non_blocking=True)
                dv[j].copy_(hv, non_blocking=True)
                in_ready[j] = ev()
                in_ready[j].record(s_in)
            stream.wait_event(in_ready[j])
            layer = i % NL
            chunk[layer] += 1
            ca.attend(layer, 0, chunk[layer], dq[j][0], dq[j][1], dq[j][2], do[j], stream)
            ca.euler(dx[j], dv[j], tm.TM_BF16, 0.5, stream)
            done = ev()
            done.record(stream)
            with torch.cuda.stream(s_out):
                s_out.wait_event(done)
                ho[j].copy_(do[j], non_blocking=True)
                hxo[j].copy_(dx[j], non_blocking=True)
                out_done[j] = ev()
                out_done[j].record(s_out)
        stream.wait_stream(s_out)
        stream.wait_stream(s_in)
        b.record(stream)
        barrier()
        e_ms = max_over_ranks(a.elapsed_time(b)) / ke
        # The host link bounds this number: time the same bytes as plain pinned
        # copies (H2D alone, then H2D and D2H concurrently) on the same streams.
        barrier()
        la, lb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        la.record(s_in)
        for _ in range(3):
            with torch.cuda.stream(s_in):
                for dst, src in zip(dq[0], hq):
                    dst.copy_(src, non_blocking=True)
                dx[0].copy_(hx, non_blocking=True)
                dv[0].copy_(hv, non_blocking=True)
        lb.record(s_in)
        barrier()
        h2d_ms = la.elapsed_time(lb) / 3
        link_ms = max_over_ranks(h2d_ms)
        e2e = {"value": flop_per_call(c) / (e_ms * 1e-3) / 1e12, "unit": "TFLOP/s",
               "ms_per_step": e_ms, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h),
               "h2d_only_ms": link_ms, "h2d_gbs": h2d / (link_ms * 1e-3) / 1e9,
               "link_bound_tflops": flop_per_call(c) / (link_ms * 1e-3) / 1e12,
               "note": "pinned host buffers, copies in the timed region, double-buffered streams; "
                       "link_bound = the step's H2D bytes alone over the measured H2D rate"}

    # ---------------------------------------------------------------- SURVEY Sec 8(f) rows,
    # the other single-GPU configs and one P = 2/4/8 rank's share: short loops,
    # measured before the long streaming run (which holds the GPU at its power
    # cap for seconds), each with the SM clocks sampled during it.
    extras = others = shards = None
    if not args.no_extras and P == 1:
        xclk = ClockSampler(local)
        xclk.start()
        x0 = time.time()
        extras = measure_extras(tm, c, torch, stream)
        x1 = time.time()
        others = measure_other_configs(tm, torch, args.config, max(10, args.steps), stream)
        x2 = time.time()
        if args.config == "wan512":
            shards = measure_shards(tm, torch, c, max(10, args.steps), stream, live_ms)
        x3 = time.time()
        xclk.stop()
        extras["clocks"] = xclk.summary(window=(x0, x1))
        others["clocks"] = xclk.summary(window=(x1, x2))
        if shards is not None:
            shards["clocks"] = xclk.summary(window=(x2, x3))

    streaming = None
    if args.stream_chunks >= 2:
        # BJ.configs[3]: chunk-by-chunk generation in the real dependency order,
        # every (layer, step) of a WAN-2.1-14B DiT (40 blocks x 2 NFE), the
        # reference cached once per (layer, step), one Euler update per step.
        NLs, NS = 40, 2
        sc = make_ctx(NLs, NS)
        for layer in range(NLs):
            for st in range(NS):
                sc.put_reference(layer, st, kref, vref, stream)
        def one_chunk(t):
            for st in range(NS):
                for layer in range(NLs):
                    q, k, v = sets[(layer + st) % NB]
                    sc.attend(layer, st, t, q, k, v, outs[layer % NB], stream)
                sc.euler(xlat, vlat, tm.TM_BF16, 1.0 / NS, stream)
        one_chunk(1)
        barrier()
        sa, sb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        sa.record(stream)
        for t in range(2, args.stream_chunks + 1):
            one_chunk(t)
        sb.record(stream)
        barrier()
        s_ms = max_over_ranks(sa.elapsed_time(sb)) / (args.stream_chunks - 1)
        if P > 1 or transport == "peer":
            sc.check()
        streaming = {"config": f"BJ.configs[3] shape: {NLs} layers x {NS} steps per chunk, "
                               f"chunks 2..{args.stream_chunks} timed (steady state, t>=2)",
                     "ms_per_chunk": s_ms,
                     "attention_calls_per_chunk": NLs * NS,
                     "tflops": NLs * NS * flop_per_call(c) / (s_ms * 1e-3) / 1e12}
        sc.close()

    fl = flop_per_call(c)
    ms_step = ms_total / args.steps
    value = fl * args.steps / (ms_total * 1e-3) / 1e12
    peak, peak_sus, peak_src = measured_peaks()
    # per GPU (each rank does 1/P of the heads); live = the attention-only loop
    achieved = fl / P / (live_ms * 1e-3) / 1e12
    achieved_alone = fl / P / (k_ms * 1e-3) / 1e12
    traffic, traffic_src = stored_traffic(args.config, P)
    cpu = None
    if rank == 0 and P == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(c, args.oracle_rows)
    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": P,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "bf16", "data": "synthetic",
            "config": {"workload": c["workload"], "heads": H, "head_dim": d, "ref_tokens": Lr,
                       "chunk_tokens": Lc, "chunk_index": ">=2", "keys_attended": Lr + 2 * Lc,
                       "gflop_per_chunk_attention": fl / 1e9, "euler_elements": c["latent"],
                       "parallelism": f"ulysses-heads{P}" if P > 1 else "single-gpu",
                       "transport": transport if (P > 1 or transport == "peer") else "none",
                       "l2": "inputs larger than L2 (8 layer caches x 4 input sets rotated)"},
            "ms_per_chunk_attention": k_ms,
            "ms_per_chunk_attention_median": k_med,
            "chunk1": {"ms": t1_ms, "keys_attended": Lr + Lc,
                       "tflops_per_gpu": flop_per_call(c, t=1) / P / (t1_ms * 1e-3) / 1e12,
                       "note": "first chunk of a stream (Lk = Lr + Lc), fused append, median of "
                               f"{NL} calls"},
            "kernel_clocks": kclk,
            "frac_of_bf16_peak": achieved / peak,
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak,
                         "unit": "TFLOP/s", "frac": achieved / peak, "traffic": traffic,
                         "traffic_source": traffic_src,
                         "kernel": "tm_fmha_sm100 (tcgen05, fused c_t append)" if P == 1 and
                                   transport == "nccl" else
                                   f"whole call ({transport} transport: exchange + attention)",
                         "timing": f"{args.steps} attention calls of the step (fused append, same "
                                   "inputs, no Euler) back to back between one CUDA event pair "
                                   "on the launching stream, right after the timed region",
                         "ms_per_launch": live_ms,
                         "peak_source": f"{peak_src} bf16 burst (MEASURED_PEAKS.json)",
                         "flop_per_launch": fl / P,
                         "algorithmic_bytes_per_launch": algo_bytes(c) / P,
                         "achieved_kernel_alone": achieved_alone,
                         "kernel_alone": "zero-copy calls (no append), per-call events, after the "
                                         "timed region" if zc else "whole calls, per-call events"},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "streaming": streaming,
            "next_rows": extras,
            "other_configs": others,
            "shards": shards,
            "gpu_launches": gpu_launches,
            "clocks": clk,
        }
        print(json.dumps(out))
    ca.close()
    if P > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
