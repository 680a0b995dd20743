#!/usr/bin/env python
"""Benchmark: SNN inference images/s on 1..8 B200 (+ NormAD training img/s).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  torchrun --nproc-per-node N --master-addr 127.0.0.1 ... bench.py --gpus N

Headline workload (BASELINE.json configs[2]): batched
inference over the 10,000 synthetic MNIST-shaped images of
synthetic_dataset(1000, seed=2000) (committed in data/workloads.npz, generated
by the reference itself), weights W_fix, T=100 ms, dt=1 ms (100 steps),
sharded contiguously over the ranks with one NCCL all-gather of the counts.
One step = the whole 10,000-image set (strong scaling).  Rank 0 also times
NormAD training (configs[1]: 1,000 images, one GPU) and, at N=1, the CPU
reference (all host cores) on a bounded sample.

--impl reference times the reference's own CPU path on the host cores: the
UNMODIFIED spikedigits package installed in baseline/_ref
(scripts/stage_reference.sh), through its public batch_counts with one worker
process per core -- or, if that install is missing, the oracle port
(oracle/snn_oracle.py, a bit-exact numpy restatement), labelled kind "port".
"""
from __future__ import annotations

import os

for _v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(_v, "1")

import argparse
import ctypes
import json
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SNN inference images/sec @1/2/4/8 B200 + NormAD train img/s, % roofline vs CPU ref"
N_IMAGES = 10_000
F_INF_PER_STEP = 389_516          # dense algorithmic flop per image-step
F_TRAIN_PER_STEP = 592_316
F_TRAIN_PER_IMAGE = 162_240
# The roofline kernel of the default configuration: the guard-band hidden
# layer k_hidden_gb<3> (hidden_gb.cuh) -- float32 pairs whose
# decisions are proven against the float64 trajectory, bound by the integer /
# logic (ALU) pipe and instruction issue.  Its work per active window-step is
# counted from the SASS of the library that runs (sass_loop_counts): the
# innermost loop is one step of TWO windows per lane (64 per warp).
HIDDEN_KERNEL = "_ZN3snn11k_hidden_gbILi3ELi20EEEvNS_9BatchArgsE"   # k_hidden_gb<3, 20>
# SASS opcodes that issue to the ALU pipe (integer / logic / compare / select)
ALU_OPS = ("LOP3", "LOP", "SHF", "ISETP", "IMNMX", "VIMNMX", "VIMNMX3", "SEL", "FSEL", "FSETP", "FMNMX", "FMNMX3",
           "IADD3", "VIADD", "LEA", "PRMT", "PLOP3", "BMSK", "FLO", "BREV", "SGXT")
FP32_FLOP = {"FFMA2": 4, "FADD2": 2, "FMUL2": 2, "FFMA": 2, "FADD": 1, "FMUL": 1}
SASS_FALLBACK = {"instructions": 237, "alu": 112, "fp32_flop": 234, "fp32_instr": 95, "windows_per_iter": 64,
                 "ops": {"LOP3": 40, "FADD2": 36, "FFMA2": 34, "ISETP": 24, "SEL": 24, "FMUL": 24, "LDS": 18,
                         "VIMNMX3": 12, "SHF": 10}}  # r02 final build, if cuobjdump is absent
LAUNCHES_PER_CHUNK = 6   # per sub-batch: k_prep, k_tile_scan, k_hidden_gb, k_hidden_fix, k_gsum, k_output
PIPE_IMAGES = 0          # snn_set_pipeline sub-batch (library default: off)


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def sass_loop_counts(so_path: str, fn: str) -> dict:
    """Opcode counts of the innermost step loop of `fn` (the smallest backward-
    branch loop with >= 20 FFMA2) in the SASS of `so_path` (cuobjdump): total
    instructions, ALU-pipe instructions (ALU_OPS), FP32 flop (FFMA2 = 4 per
    lane ...).  Falls back to SASS_FALLBACK (source: "fallback")."""
    import collections
    import re
    import shutil
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    try:
        txt = subprocess.run([tool, "-sass", "-fun", fn, so_path], capture_output=True, text=True,
                             timeout=120).stdout.split("\n")
    except (OSError, subprocess.TimeoutExpired):
        txt = []
    ins = []
    for line in txt:
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m:
            ins.append((int(m.group(1), 16), m.group(2)))
    best = None
    for a, t in ins:
        m = re.search(r"BRA(?:\.\w+)* (?:!?U?P[T\d], )?(0x[0-9a-f]+)", t)
        if not m or int(m.group(1), 16) >= a:
            continue
        body = [x for x in ins if int(m.group(1), 16) <= x[0] <= a]
        cnt = collections.Counter((tt.split()[1] if tt.startswith("@") else tt.split()[0]).split(".")[0]
                                  for _, tt in body)
        if cnt["FFMA2"] >= 20 and (best is None or len(body) < best["instructions"]):
            best = {"instructions": len(body), "alu": sum(cnt[o] for o in ALU_OPS),
                    "fp32_flop": sum(cnt[o] * f for o, f in FP32_FLOP.items()),
                    "fp32_instr": sum(cnt[o] for o in FP32_FLOP), "windows_per_iter": 64,
                    "ops": dict(cnt.most_common(12))}
    if best is None:
        return dict(SASS_FALLBACK, source="fallback (cuobjdump unavailable)")
    return dict(best, source=f"cuobjdump -sass -fun {fn} {os.path.basename(so_path)}")


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class Clocks:
    """SM clock + throttle-reason sampler running during the timed region
    (B200_PROFILING.md clocks line).  NVML every 2 ms (the timed region of a
    step is only a few ms); nvidia-smi -lms 100 if NVML is unavailable."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap"}
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.nv = None
        self.lines = []
        self.sm, self.mask, self.max = [], 0, None
        self.stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[self.index]) if vis and vis.split(",")[self.index].strip().isdigit() else self.index
            self.h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.max = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
            self.nv = pynvml
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            return self
        except Exception:
            self.nv = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _poll(self):
        nv = self.nv
        while not self.stop.is_set():
            try:
                self.sm.append(float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)))
                self.mask |= int(nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            except Exception:
                pass
            time.sleep(0.002)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        self.stop.set()
        if self.nv is not None:
            self.t.join(timeout=1)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        if self.nv is not None:
            reasons = sorted(n for b, n in self.REASONS.items() if self.mask & b)
            return {"sm_mhz": statistics.median(self.sm) if self.sm else None, "sm_max_mhz": self.max,
                    "reasons": reasons, "samples": len(self.sm), "source": "nvml, 2 ms period"}
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for name, val in zip(names, f[5:9]):
                if val.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm), "source": "nvidia-smi -lms 100"}


def measure_peaks():
    """FP64 DFMA / FP32 FFMA (TFLOP/s) and ALU LOP3 (Tops, lane ops) peaks of
    this GPU (libsnn_peaks.so microbenchmarks), best of 3."""
    from paper_1711_03637_b200.build import PEAKS_OUT
    lib = ctypes.CDLL(PEAKS_OUT)
    f64, f32, alu = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    best64 = best32 = bestalu = 0.0
    for _ in range(3):
        lib.snn_measure_fma_peaks(ctypes.byref(f64), ctypes.byref(f32))
        lib.snn_measure_alu_peak(ctypes.byref(alu))
        best64, best32, bestalu = max(best64, f64.value), max(best32, f32.value), max(bestalu, alu.value)
    return best64, best32, bestalu


def active_positions(images: np.ndarray) -> np.ndarray:
    """Windows with any non-zero pixel, per image (the ones k_hidden simulates)."""
    nz = images.reshape(-1, 28, 28) != 0
    win = np.zeros((len(images), 26, 26), dtype=bool)
    for a in range(3):
        for b in range(3):
            win |= nz[:, a:a + 26, b:b + 26]
    return win.reshape(len(images), -1).sum(axis=1)


def load_workload():
    d = np.load(os.path.join(ROOT, "data", "workloads.npz"))
    w = np.load(os.path.join(ROOT, "data", "w_fix.npz"))["w_fix"]
    return d, w


# ============================================================== reference arm
REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def stock_reference():
    """The unmodified reference (pip-installed in baseline/_ref by
    scripts/stage_reference.sh): (batch_counts, train_epoch, NetworkConfig,
    default_filter_bank, LearnConfig) from its own modules, or None."""
    if not os.path.isdir(os.path.join(REF_DIR, "spikedigits")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    try:
        from spikedigits.evaluate import batch_counts
        from spikedigits.filters import default_filter_bank
        from spikedigits.network import NetworkConfig
        from spikedigits.normad import LearnConfig, train_epoch
    except Exception as e:  # noqa: BLE001 -- report and fall back to the port
        log(f"[reference] stock reference not importable ({e}); timing the oracle port")
        return None
    assert "baseline" in sys.modules["spikedigits"].__file__
    return batch_counts, train_epoch, NetworkConfig, default_filter_bank, LearnConfig


def reference_infer(imgs, w, cores):
    """(callable(images) -> counts, kind, description) of the reference's CPU
    batched inference on `cores` worker processes."""
    ref = stock_reference()
    if ref is not None:
        bc, _, NC, bank, _ = ref
        cfg, fb = NC(), bank()
        return (lambda x: bc(x, w, fb, cfg, workers=cores)), "reference", \
            f"stock spikedigits.evaluate.batch_counts(workers={cores}) from baseline/_ref"
    from oracle import snn_oracle as orc
    p = orc.Params()
    return (lambda x: orc.batch_counts(x, w, p, workers=cores)), "port", \
        f"oracle.batch_counts(workers={cores}) (bit-exact port)"


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    d, w = load_workload()
    imgs = d["c3_images"]
    cores = host_cores()
    sample = int(min(len(imgs), max(2 * cores, cores * 32)))
    fn, kind, desc = reference_infer(imgs, w, cores)
    log(f"[reference] {desc}, {sample} images per step")
    for _ in range(args.warmup):
        fn(imgs[:sample])
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        got = fn(imgs[:sample])
        times.append(time.perf_counter() - t0)
    ref10k = np.load(os.path.join(ROOT, "tests", "golden", "c3_counts_reference.npz"))["counts"]
    value = sample * len(times) / sum(times)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "images/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (reference strokes generator)",
        "config": {"workload": "c3 batched inference (reference CPU path), bounded sample",
                   "n_images_per_step": sample, "t_ms": 100.0, "dt_ms": 1.0, "n_steps": 100,
                   "parallelism": f"{cores} host processes"},
        "cpu_baseline": {"value": value, "unit": "images/s", "cores": cores, "kind": kind,
                         "sample": f"first {sample} of the 10,000 c3 images per step, {desc}, {cpu_model()}"},
        "e2e": {"value": value, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "counts_equal_committed_reference_counts": bool(np.array_equal(got, ref10k[:sample])),
    }
    print(json.dumps(line), flush=True)


# ============================================================== our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1711_03637_b200 as sd
    from paper_1711_03637_b200 import distributed as sdist
    from paper_1711_03637_b200.engine import get_engine, make_consts

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # test-only overrides (SNN_BENCH_DEVICE / SNN_BENCH_BACKEND): run several
    # ranks on one GPU over gloo to exercise the multi-rank path on a 1-GPU box
    local = int(os.environ.get("SNN_BENCH_DEVICE", local))
    torch.cuda.set_device(local)
    if world > 1:
        backend = os.environ.get("SNN_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(vals):
        t = torch.tensor(vals, dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.tolist()

    d, w_fix = load_workload()
    imgs_all = d["c3_images"]
    cfg, bank = sd.NetworkConfig(), sd.default_filter_bank()
    c = make_consts(cfg, bank)
    eng = get_engine()
    a, b = sdist.shard_bounds(N_IMAGES, world)[rank]
    shard = imgs_all[a:b].reshape(b - a, -1)
    with torch.cuda.stream(eng.stream):
        d_img = torch.from_numpy(shard.copy()).to(eng.device)
        d_w = torch.from_numpy(w_fix.copy()).to(eng.device)
        flush = torch.empty(256 << 20, dtype=torch.uint8, device=eng.device)
    eng.stream.synchronize()
    per_img_ws = eng.lib.snn_infer_workspace(ctypes.byref(c), 1)
    chunk = max(1, min(b - a, (4 << 30) // per_img_ws))
    chunks_per_step = -(-(b - a) // chunk)
    launches_per_step = LAUNCHES_PER_CHUNK * chunks_per_step

    def step():
        out = eng.infer(c, d_img, d_w)["counts"]
        with torch.cuda.stream(eng.stream):
            return sdist.gather_counts(out, N_IMAGES) if world > 1 else out

    for _ in range(args.warmup):
        step()
    eng.stream.synchronize()
    barrier()

    # The K calls are enqueued back to back (no host sync between them, as a
    # serving loop would issue them), so the host's per-call launch work
    # overlaps the previous call instead of idling the GPU inside a step.
    evs = []
    with Clocks(local) as clk:
        torch.cuda.synchronize()
        barrier()
        for _ in range(args.steps):
            with torch.cuda.stream(eng.stream):
                flush.zero_()               # evict the 7.8 MB input set from the 126 MB L2
            e0, k1, e1 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            e0.record(eng.stream)
            out = eng.infer(c, d_img, d_w)["counts"]
            k1.record(eng.stream)
            if world > 1:
                with torch.cuda.stream(eng.stream):
                    out = sdist.gather_counts(out, N_IMAGES)
            e1.record(eng.stream)
            evs.append((e0, k1, e1))
        torch.cuda.synchronize()
        barrier()
    step_ms = [e0.elapsed_time(e1) for e0, _, e1 in evs]
    kern_ms = [e0.elapsed_time(k1) for e0, k1, _ in evs]
    clocks = clk.summary()
    tot_ms, ker_ms = max_over_ranks([sum(step_ms), sum(kern_ms)])
    # roofline pass: k_hidden timed alone (one un-pipelined launch per call,
    # CUDA events the library records around it on its stream)
    hk_ms, call1_ms = kernel_alone_ms(eng, c, d_img, d_w, flush, args.steps)
    stage_ms = stage_times(eng, c, d_img, d_w, flush, args.steps)
    value = N_IMAGES * args.steps / (tot_ms / 1e3)
    counts_dev = out
    ref_prefix = None
    if rank == 0:
        gold = np.load(os.path.join(ROOT, "tests", "golden", "reference_golden.npz"))["c3_counts_200"]
        ref_prefix = bool(np.array_equal(counts_dev[:200].cpu().numpy(), gold)) if counts_dev.shape[0] >= 200 else None
    ref_all = None
    if rank == 0 and counts_dev.shape[0] == N_IMAGES:  # all 10,000 (gathered) vs the reference's own batch_counts
        ref10k = np.load(os.path.join(ROOT, "tests", "golden", "c3_counts_reference.npz"))["counts"]
        ref_all = bool(np.array_equal(counts_dev.cpu().numpy(), ref10k))
    # near-tie accounting (untimed): output steps of this shard whose threshold
    # decision could differ from the reference's under the rounding bound of
    # the reordered c_hidden @ W (snn_infer_out_t.near_ties)
    tie_out = eng.infer(c, d_img, d_w, ties=True)
    eng.stream.synchronize()
    near_ties = torch.tensor([float(tie_out["near_ties"].sum().item())], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(near_ties, op=dist.ReduceOp.SUM)
    near_ties = near_ties.item()
    plain_out = eng.infer(c, d_img, d_w)
    ties_counts_same = bool(torch.equal(tie_out["counts"], plain_out["counts"]))
    hidden_redo = int(plain_out["hidden_redo"].item())
    hidden_frac = hidden_per_neuron_frac(eng, c, imgs_all, w_fix) if rank == 0 else None

    # ---- e2e: public API with host buffers (H2D images + weights, D2H counts)
    e2e_times = []
    for i in range(args.warmup + args.steps):
        barrier()
        t0 = time.perf_counter()
        res = sdist.sharded_batch_counts(imgs_all, w_fix, bank, cfg)
        dt_s = time.perf_counter() - t0
        if i >= args.warmup:
            e2e_times.append(dt_s)
    (e2e_s,) = max_over_ranks([sum(e2e_times)])
    e2e_value = N_IMAGES * args.steps / e2e_s
    h2d = (b - a) * 784 + w_fix.nbytes
    d2h = N_IMAGES * 10 * 4

    line = None
    if rank == 0:
        f64, f32, alu_peak = measure_peaks()
        act = active_positions(shard.reshape(-1, 28, 28))
        n_steps = c.n_steps
        assert chunks_per_step == 1, "k_hidden events time one launch per step"
        call_ms = ker_ms / args.steps                        # whole (pipelined) snn_infer call
        from paper_1711_03637_b200 import _native
        sass = sass_loop_counts(_native.LIB_PATH, HIDDEN_KERNEL)
        gb_ms = stage_ms.get("k_hidden_gb")
        launch_ms = gb_ms if gb_ms else hk_ms                # k_hidden_gb alone (live CUDA events)
        warp_steps = float(act.sum()) * n_steps / sass["windows_per_iter"]
        alu_tops = warp_steps * sass["alu"] * 32 / (launch_ms * 1e-3) / 1e12
        fp32_tflops = warp_steps * sass["fp32_flop"] * 32 / (launch_ms * 1e-3) / 1e12
        clk_ghz = (clocks.get("sm_mhz") or 1965.0) / 1e3
        issue_frac = warp_steps * sass["instructions"] / (launch_ms * 1e-3) / (4 * torch.cuda.get_device_properties(0).multi_processor_count * clk_ghz * 1e9)
        dense_tflops = (b - a) * F_INF_PER_STEP * n_steps / (ker_ms / args.steps * 1e-3) / 1e12
        traffic_bytes, traffic_src = committed_traffic("k_hidden_gb")
        line = {
            "metric": METRIC, "value": value, "unit": "images/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot_ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: reference stroke generator images (data/workloads.npz), reference-trained W_fix",
            "config": {"workload": "c3: batched inference, 10,000 synthetic MNIST-shaped 28x28 images, "
                                   "12x3x3 feature maps (8112 LIF) -> 10 LIF, T=100 ms, dt=1 ms",
                       "n_images": N_IMAGES, "t_ms": 100.0, "dt_ms": 1.0, "n_steps": n_steps,
                       "parallelism": f"dp{world}", "collective": (f"one all_gather of int32 counts "
                                                                    f"({dist.get_backend()})") if world > 1 else "none",
                       "l2": "flushed between timed steps (256 MiB write)"},
            "e2e": {"value": e2e_value, "unit": "images/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h), "api": "distributed.sharded_batch_counts (host numpy in/out)"},
            "gpu_launches": int(args.steps * launches_per_step),
            "roofline": {"bound": "alu", "achieved": alu_tops, "peak": alu_peak, "unit": "Tops (int32 lane ops)",
                         "frac": alu_tops / alu_peak, "traffic": traffic_bytes,
                         "traffic_unit": "bytes per launch (DRAM read + write)", "traffic_source": traffic_src,
                         "kernel": "k_hidden_gb<3>: fused input-table gather + 3x3 stencil + hidden LIF in float32 "
                                   "pairs with a per-window float64 error band (windows near a threshold decision "
                                   "re-simulated in float64 by k_hidden_fix), spike raster out; timed alone with "
                                   "the library's live CUDA events (snn_profile_stage_events)",
                         "achieved_basis": f"ALU-pipe lane ops executed: active windows ({int(act.sum())}) x N "
                                           f"({n_steps}) / {sass['windows_per_iter']} windows per warp-iteration x "
                                           f"{sass['alu']} ALU instructions x 32 lanes (inner loop of "
                                           f"{sass['instructions']} SASS instructions: {sass['ops']}; "
                                           f"{sass['source']})",
                         "peak_source": "measured in this run: LOP3 throughput microbenchmark (libsnn_peaks.so); "
                                        "MEASURED_PEAKS.json has no integer-pipe figure",
                         "launch_ms": launch_ms, "hidden_layer_ms": hk_ms, "call_ms": call_ms,
                         "unpipelined_call_ms": call1_ms,
                         "issue_frac": issue_frac,
                         "issue_basis": f"{sass['instructions']} SASS instructions per warp-iteration against 4 "
                                        f"issue slots per SM per cycle at the sampled SM clock ({clk_ghz:.3f} GHz)",
                         "fp32_tflops": fp32_tflops, "fp32_peak_tflops": f32, "fp32_frac": fp32_tflops / f32,
                         "fp32_basis": f"{sass['fp32_flop']} FP32 flop per warp-iteration per lane "
                                       f"({sass['fp32_instr']} FFMA2/FADD2/FMUL2/FMUL.SAT)",
                         "fp64_peak_tflops": f64,
                         "dense_equiv_tflops": dense_tflops,
                         "dense_equiv_basis": "SURVEY 8(d) F_inf = 389,516 flop per image-step over the whole call",
                         "active_windows_per_image": float(act.mean()),
                         "kernels": kernel_table(stage_ms, call1_ms, alu_tops / alu_peak)},
            "clocks": clocks,
            "parity": {"c3_first200_counts_equal_reference": ref_prefix,
                       "c3_all10000_counts_equal_reference": ref_all,
                       "hidden_per_neuron_counts_equal_frac": hidden_frac,
                       "hidden_per_neuron_basis": "1,000 c3 images x 8,112 neurons vs the reference's forward_pass "
                                                  "(tests/golden/c3_hidden_counts_reference.npz)",
                       "output_near_ties": int(near_ties),
                       "output_near_ties_basis": "output steps within the rigorous rounding bound of the "
                                                 "reordered c_hidden @ W, all 10,000 c3 images (0 = counts "
                                                 "provably the reference's)",
                       "counts_with_tie_detector_unchanged": ties_counts_same,
                       "hidden_redo_windows": hidden_redo,
                       "hidden_redo_basis": "windows of the 10,000 images whose float32 trajectory came within "
                                            "the error band of a threshold decision and were re-simulated in "
                                            "float64 (k_hidden_fix); the raster is the float64 kernel's "
                                            "bit for bit (tests/test_gpu_round2.py)"},
        }
    # ---- NormAD training (single GPU, rank 0)
    if rank == 0 and not args.skip_train:
        line["train"] = bench_train(args, sd, eng, d, cfg, bank)
    if rank == 0 and not args.skip_latency:
        line["latency"] = bench_latency(sd, d, w_fix, bank)
        line["preprocess"] = bench_preprocess(sd, w_fix, bank)
    if rank == 0 and world == 1 and not args.skip_cpu:
        line["cpu_baseline"] = cpu_baseline(d, w_fix)
    if rank == 0 and not args.skip_c5 and os.path.exists(os.path.join(ROOT, "data", "c5_workload.npz")):
        line["full_pass"] = bench_c5(sd, eng, cfg, bank, line)
    if rank == 0:
        print(json.dumps(line), flush=True)
    barrier()
    if world > 1:
        dist.destroy_process_group()


def hidden_per_neuron_frac(eng, c, imgs_all, w):
    """Fraction of the 1,000 reference images (every 10th c3 image) whose
    8,112 per-neuron hidden spike counts equal the reference's forward_pass
    (tests/golden/c3_hidden_counts_reference.npz), from the GPU raster."""
    import torch
    from paper_1711_03637_b200.api import decode_hidden
    gp = os.path.join(ROOT, "tests", "golden", "c3_hidden_counts_reference.npz")
    if not os.path.exists(gp):
        return None
    g = np.load(gp)
    imgs = imgs_all[g["idx"]].reshape(len(g["idx"]), -1)
    with torch.cuda.stream(eng.stream):
        d_img = torch.from_numpy(imgs.copy()).to(eng.device)
        d_w = torch.from_numpy(w.copy()).to(eng.device)
    out = eng.infer(c, d_img, d_w, raster=True)
    eng.stream.synchronize()
    raster = out["raster"].cpu().numpy()
    tpos, nt, tb = out["tile_pos"].cpu().numpy(), out["n_tiles"].cpu().numpy(), out["tile_base"].cpu().numpy()
    same = 0
    for i in range(len(imgs)):
        h = decode_hidden(raster, int(tb[i]), tpos[i], int(nt[i]), c.n_steps)
        same += int(np.array_equal(h.sum(axis=0), g["hidden_counts"][i]))
    return same / len(imgs)


def stage_times(eng, c, d_img, d_w, flush, steps):
    """Per-kernel device time of a live un-pipelined snn_infer call: CUDA
    events the library records between its launches on its stream
    (snn_profile_stage_events; event 6 between the guard-band hidden kernel
    and its float64 redo), L2 flushed before each call; medians."""
    import torch
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(7)]
    for e in evs:
        e.record(eng.stream)   # created lazily on first record
    arr = (ctypes.c_void_p * 7)(*[e.cuda_event for e in evs])
    per = {}
    try:
        for _ in range(max(3, steps)):
            with torch.cuda.stream(eng.stream):
                flush.zero_()
            evs[6].record(eng.stream)  # stays before k_prep when no guard-band launch re-records it
            eng.lib.snn_profile_stage_events(arr, 7)
            eng.infer(c, d_img, d_w)
            eng.lib.snn_profile_stage_events(None, 0)
            evs[5].synchronize()
            t = [0.0] + [evs[0].elapsed_time(evs[k]) for k in range(1, 7)]
            gb = t[6] > t[2]
            st = {"k_prep": t[1], "k_tile_scan": t[2] - t[1]}
            if gb:
                st.update({"k_hidden_gb": t[6] - t[2], "k_hidden_fix": t[3] - t[6]})
            else:
                st["k_hidden_res"] = t[3] - t[2]
            st.update({"k_gsum": t[4] - t[3], "k_output": t[5] - t[4]})
            for k, v in st.items():
                per.setdefault(k, []).append(v)
    finally:
        eng.lib.snn_profile_stage_events(None, 0)
    return {k: statistics.median(v) for k, v in per.items()}


def committed_kernels():
    """Per-kernel ncu metrics of the newest committed capture
    (profiles/<round>_kernels.json, scripts/summarize_profiles.py)."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*_kernels.json")))
    if not files:
        return {}, None
    return json.load(open(files[-1])), os.path.relpath(files[-1], ROOT)


def _short(name: str) -> str:
    return name.split("(")[0].split("<")[0].split()[-1].split("::")[-1]


def kernel_table(stage_ms, call_ms, hidden_frac):
    """Every kernel of the inference call: live duration (CUDA events) and its
    share of the call, the bound that limits it and the fraction of that bound
    -- the FP64 flop fraction for the hidden layer (measured here), the
    committed ncu capture's pipe / issue / DRAM figures for the rest."""
    prof, src = committed_kernels()
    ncu = {}
    for name, recs in prof.items():
        ncu.setdefault(_short(name), recs[0])
    mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    hbm = float(mp.get("hbm_gbs", 6553.3))
    bounds = {"k_prep": "hbm/latency (one pass over the images)", "k_tile_scan": "latency (one CTA)",
              "k_hidden_gb": "ALU pipe / issue (float32 pairs + integer decisions)",
              "k_hidden_fix": "fp64 dependent chain per flagged window (latency)",
              "k_hidden_res": "fp64 pipe", "k_gsum": "L1 data pipe / issue (step lists, W-row gathers)",
              "k_output": "fp64 dependent chain per image (latency)"}
    out = {}
    for k, ms in stage_ms.items():
        e = {"ms": ms, "share_of_call": ms / call_ms if call_ms else None, "bound": bounds.get(k)}
        n = ncu.get(k) or ncu.get({"k_output": "k_output_dist", "k_hidden_fix": "k_hidden_fix_res"}.get(k, ""))
        if n:
            e["ncu"] = {x: n.get(x) for x in ("issue_active_pct", "fp64_pipe_pct", "alu_pipe_pct", "fma_pipe_pct",
                                              "dram_bytes", "duration_ms") if n.get(x) is not None}
            if n.get("dram_bytes"):
                e["dram_frac_of_hbm_peak"] = n["dram_bytes"] / (ms * 1e-3) / 1e9 / hbm
        if k == "k_hidden_gb":
            e["frac"] = hidden_frac
            e["frac_basis"] = "executed ALU-pipe lane ops / LOP3 peak (roofline.frac)"
            if n and n.get("alu_pipe_pct") is not None:
                e["ncu_alu_pipe_frac"] = n["alu_pipe_pct"] / 100.0
        elif k == "k_gsum" and n:
            iss, l1 = (n.get("issue_active_pct") or 0) / 100.0, (n.get("l1_wavefronts_pct") or 0) / 100.0
            e["frac"] = max(iss, l1)
            e["bound"] = ("L1 data pipe (step-list and W-row gather wavefronts)" if l1 >= iss
                          else "issue (list building, W-row gathers)")
            e["frac_basis"] = ("the busier of the L1 data-pipe wavefronts and the issue slots (ncu); DRAM is "
                               "dram_frac_of_hbm_peak")
        elif k == "k_output" and n:
            fp, iss = (n.get("fp64_pipe_pct") or 0) / 100.0, (n.get("issue_active_pct") or 0) / 100.0
            l1 = (n.get("l1_wavefronts_pct") or 0) / 100.0
            e["frac"] = max(fp, iss, l1)
            e["bound"] = ("L1 data pipe (the lane-distributed step's candidate exchange, k_output_dist)" if l1 >= max(fp, iss)
                          else "issue (lane-distributed step, k_output_dist)" if iss >= fp else "fp64 pipe")
            e["frac_basis"] = ("the busiest of the L1 data pipe, the FP64 pipe and the issue slots (ncu); a warp is "
                               "one image's serial chain")
        elif n:
            e["frac"] = (n.get("issue_active_pct") or 0) / 100.0
            e["frac_basis"] = "issue slots busy (ncu)"
        out[k] = e
    out["_source"] = f"live CUDA events (snn_profile_stage_events) + {src or 'no committed ncu capture'}"
    return out


def kernel_alone_ms(eng, c, d_img, d_w, flush, steps):
    """k_hidden alone: pipelining off (one k_hidden launch per call), CUDA
    events recorded by the library around the launch (snn_profile_events);
    returns (k_hidden ms, un-pipelined call ms), medians over `steps` calls."""
    import torch
    lib = eng.lib
    lib.snn_set_pipeline(0, 0)
    ev_b, ev_a = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev_b.record(eng.stream)   # torch creates the CUDA events lazily, on first record
    ev_a.record(eng.stream)
    hk, call = [], []
    try:
        eng.infer(c, d_img, d_w)
        for _ in range(max(3, steps)):
            with torch.cuda.stream(eng.stream):
                flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(eng.stream)
            lib.snn_profile_events(ctypes.c_void_p(ev_b.cuda_event), ctypes.c_void_p(ev_a.cuda_event))
            eng.infer(c, d_img, d_w)
            lib.snn_profile_events(None, None)
            e1.record(eng.stream)
            e1.synchronize()
            hk.append(ev_b.elapsed_time(ev_a))
            call.append(e0.elapsed_time(e1))
    finally:
        lib.snn_profile_events(None, None)
        lib.snn_set_pipeline(PIPE_IMAGES, 0)
    return statistics.median(hk), statistics.median(call)


def committed_traffic(prefix):
    """DRAM bytes per launch of the roofline kernel from the newest committed
    ncu --set full capture (profiles/<round>_traffic.json, written by
    scripts/summarize_profiles.py); (None, None) when there is none."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*_traffic.json")))
    if not files:
        return None, None
    data = json.load(open(files[-1]))
    for name, recs in data.items():
        if name.split("<")[0].split("::")[-1].strip().split()[-1].startswith(prefix) and recs:
            r = recs[0]
            return r["dram_bytes"], (f"{os.path.relpath(files[-1], ROOT)}: {name}, {r['capture']} "
                                     f"(ncu --set full, 10,000-image launch, read {r['dram_read_bytes']:.3g} B + "
                                     f"write {r['dram_write_bytes']:.3g} B)")
    return None, None


def train_chunks(eng, c, n):
    """Chunks of one snn_train call (a 64-image first chunk, then full ones)."""
    chunk = int(eng.lib.snn_train_chunk(ctypes.byref(c), n))
    if n <= chunk:
        return 1
    first = min(chunk, 64)
    return 1 + -(-(n - first) // chunk)


def train_launches(eng, c, n):
    """Kernel launches of one snn_train call: per chunk k_prep, k_tile_scan,
    the hidden layer (guard band + redo for chunks of >= 256 images, else the
    float64 kernel), k_compact, k_shard, the NormAD kernel."""
    chunk = int(eng.lib.snn_train_chunk(ctypes.byref(c), n))
    sizes = [n] if n <= chunk else [min(chunk, 64)]
    while sum(sizes) < n:
        sizes.append(min(chunk, n - sum(sizes)))
    return sum(7 if s >= 256 else 6 for s in sizes)


def critical_path_model(c):
    """Per-image latency floor of the sequential NormAD chain (DESIGN.md 4,
    4.1): the output scan's dependent chain per step (no output spike: 6 FP64
    ops of 8.2 cycles + threshold test, ballot and select ~25 cycles; after an
    output spike, 23% of steps, + bumps, difference and the 5-level pairwise
    sum: 8 more FP64 ops) at the max SM clock.  In the speculative kernel (the
    default) the R adjoint, dW, the partial sums and the proof bound run on
    the other warps under the next image's scan, so the chain is the scan;
    cluster barriers and the check are not counted.  Latencies from
    scripts/scan_micro.py (FP64 dependent op 8.2 cycles)."""
    n = c.n_steps
    lat = 8.2
    scan = 0.77 * (6 * lat + 25) + 0.23 * (14 * lat + 25)
    adj = 2 * lat
    cyc = n * scan
    scan_meas = 228.0  # cycles per step of the speculative scan, clock-stamped (scripts/scan_stamps.py)
    return {"model_us_per_image": cyc / 1965.0, "scan_cycles_per_step": scan,
            "adjoint_cycles_per_step_off_chain": adj, "n_steps": n, "clock_mhz": 1965,
            "scan_measured_cycles_per_step": scan_meas, "scan_measured_us_per_image": n * scan_meas / 1965.0,
            "basis": "dependent-chain latency only (FP64 8.2 cycles); measured scan: 228 cycles/step, issue-bound "
                     "single warp of ~160 instructions per step (scripts/scan_stamps.py)"}


def train_kernel_table():
    """The training kernels' bounds and the fraction of each, from the newest
    committed ncu capture (profiles/<round>_kernels.json): k_normad_spec (or
    k_normad_cl when the speculative kernel is off) is the sequential chain (its fraction is the dependent-chain model over the
    measured time per image, critical_path.frac_of_measured); k_compact and
    k_shard are the W-independent preparation, overlapped with the chain on
    an auxiliary stream (issue slots busy)."""
    prof, src = committed_kernels()
    out = {}
    for name, recs in prof.items():
        k = _short(name)
        if k in ("k_compact", "k_shard", "k_normad_cl", "k_normad_spec"):
            r = recs[0]
            e = {"ncu": {x: r.get(x) for x in ("duration_ms", "issue_active_pct", "fp64_pipe_pct", "alu_pipe_pct",
                                              "dram_bytes") if r.get(x) is not None}}
            if k == "k_normad_spec":
                e["bound"] = ("latency: one-warp output scan per image (8 of 148 SMs); the update of the "
                              "previous image runs under it on the other warps")
                e["frac_basis"] = "critical_path.frac_of_measured"
            elif k == "k_normad_cl":
                e["bound"] = "latency: one-warp output scan + adjoint recursion per image (8 of 148 SMs)"
                e["frac_basis"] = "critical_path.frac_of_measured"
            else:
                e["bound"] = "issue / latency (per-image compaction, overlapped with the chain)"
                e["frac"] = (r.get("issue_active_pct") or 0) / 100.0
                e["frac_basis"] = "issue slots busy (ncu)"
            out[k] = e
    out["_source"] = src
    return out


def bench_train(args, sd, eng, d, cfg, bank):
    import torch
    from paper_1711_03637_b200.engine import make_consts
    learn = sd.LearnConfig()
    order = d["c2_order"]
    imgs = d["c2_images"][order].reshape(len(order), -1)
    labs = d["c2_labels"][order].astype(np.uint8)
    c = make_consts(cfg, bank, learn)
    with torch.cuda.stream(eng.stream):
        d_img = torch.from_numpy(imgs.copy()).to(eng.device)
        d_lab = torch.from_numpy(labs.copy()).to(eng.device)
        d_w = torch.zeros((8112, 10), dtype=torch.float64, device=eng.device)
    eng.train(c, d_img, d_lab, d_w)
    times = []
    for _ in range(max(2, min(args.steps, 3))):
        d_w.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(eng.stream)
        _, status = eng.train(c, d_img, d_lab, d_w)
        e1.record(eng.stream)
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
    n = len(order)
    value = n / (statistics.median(times) / 1e3)
    wf = np.load(os.path.join(ROOT, "data", "w_fix.npz"))["w_fix"]
    rel = float(np.abs(d_w.cpu().numpy() - wf).max() / np.abs(wf).max())
    # e2e: train_epoch API from host arrays (images, labels and weights H2D,
    # weights and counts D2H included); two untimed calls, median of five
    e2e_t = []
    # the caller's shuffled arrays and zero weights exist before the call
    ord_img, ord_lab = np.ascontiguousarray(d["c2_images"][order]), np.ascontiguousarray(d["c2_labels"][order])
    for rep in range(7):
        w0 = sd.zero_weights()
        t0 = time.perf_counter()
        w_api, stats = sd.train_epoch(ord_img, ord_lab, w0, bank, cfg, learn)
        if rep >= 2:
            e2e_t.append(time.perf_counter() - t0)
    e2e = n / statistics.median(e2e_t)
    # CPU reference: the stock reference's train_epoch (one process, as it trains) on 30 images
    k = 30
    ref = stock_reference()
    if ref is not None:
        _, te, NC, fb, LC = ref
        t0 = time.perf_counter()
        te(d["c2_images"][order][:k], d["c2_labels"][order][:k], np.zeros((8112, 10)), fb(), NC(), LC())
        kind, desc = "reference", f"stock spikedigits.normad.train_epoch on the first {k} images (1 process)"
    else:
        from oracle import snn_oracle as orc
        t0 = time.perf_counter()
        orc.train_epoch(d["c2_images"][order][:k], d["c2_labels"][order][:k], np.zeros((8112, 10)), orc.Params())
        kind, desc = "port", f"oracle.train_epoch on the first {k} images (1 core, as the reference)"
    cpu = k / (time.perf_counter() - t0)
    return {"metric": "NormAD online training images/s (1 GPU, sequential)", "value": value, "unit": "images/s",
            "workload": "c2: 1,000 synthetic images in epoch_permutation(0,0,1000) order from zero weights, "
                        "T=100 ms, dt=1 ms, lr=2e-7", "ms_per_epoch": statistics.median(times),
            "e2e": {"value": e2e, "unit": "images/s", "api": "train_epoch (host numpy in/out)"},
            "w_rel_err_vs_reference_epoch": rel, "train_errors": stats.n_errors,
            "dense_equiv_tflops": value * (F_TRAIN_PER_STEP * 100 + F_TRAIN_PER_IMAGE) / 1e12,
            "gpu_launches_per_epoch": train_launches(eng, c, n),
            "critical_path": dict(critical_path_model(c), frac_of_measured=critical_path_model(c)[
                "model_us_per_image"] / (statistics.median(times) * 1e3 / n),
                scan_share_of_measured=critical_path_model(c)["scan_measured_us_per_image"] /
                (statistics.median(times) * 1e3 / n)),
            "kernels": train_kernel_table(),
            "cpu_baseline": {"value": cpu, "unit": "images/s", "cores": 1, "kind": kind, "sample": desc}}


def bench_c5(sd, eng, cfg, bank, line):
    """BASELINE configs[4] / SURVEY 8(d) config 5: one NormAD pass over the
    60,000 images of synthetic_dataset(6000, seed=4000) in
    epoch_permutation(0, 0, 60000) order from zero weights, then evaluation of
    the 10,000 images of synthetic_dataset(1000, seed=5000) -- device time of
    the whole pass (one training call + one inference call), and end to end
    through train_epoch + batch_counts with host arrays.  Checked against the
    reference's own run of the same pass (tests/golden/c5_reference.npz)."""
    import torch
    from paper_1711_03637_b200.engine import make_consts
    d5 = np.load(os.path.join(ROOT, "data", "c5_workload.npz"))
    order = d5["order"]
    tr = d5["train_images"][order]
    lab = d5["train_labels"][order]
    ev = d5["eval_images"]
    learn = sd.LearnConfig()
    ct, ci = make_consts(cfg, bank, learn), make_consts(cfg, bank)
    with torch.cuda.stream(eng.stream):
        d_tr = torch.from_numpy(tr.reshape(len(tr), -1).copy()).to(eng.device)
        d_lab = torch.from_numpy(lab.astype(np.uint8)).to(eng.device)
        d_ev = torch.from_numpy(ev.reshape(len(ev), -1).copy()).to(eng.device)
        d_w = torch.zeros((8112, 10), dtype=torch.float64, device=eng.device)
    eng.train(ct, d_tr[:1000], d_lab[:1000], d_w)          # warm-up (workspaces, tables)
    eng.infer(ci, d_ev[:1000], d_w)
    d_w.zero_()
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record(eng.stream)
    counts_tr, status = eng.train(ct, d_tr, d_lab, d_w)
    e1.record(eng.stream)
    counts_ev = eng.infer(ci, d_ev, d_w)["counts"]
    e2.record(eng.stream)
    e2.synchronize()
    t_train, t_eval = e0.elapsed_time(e1) / 1e3, e1.elapsed_time(e2) / 1e3
    w = d_w.cpu().numpy()
    ctr, cev = counts_tr.cpu().numpy(), counts_ev.cpu().numpy()
    n_tr, n_ev = len(tr), len(ev)
    # end to end through the public API (host arrays in and out)
    t0 = time.perf_counter()
    w_api, stats = sd.train_epoch(tr, lab, sd.zero_weights(), bank, cfg, learn)
    cev_api = sd.batch_counts(ev, w_api, bank, cfg)
    e2e_s = time.perf_counter() - t0
    out = {"metric": "full NormAD pass (60,000 train) + 10,000-image eval, images/s (1 GPU)",
           "value": (n_tr + n_ev) / (t_train + t_eval), "unit": "images/s",
           "train_images_per_s": n_tr / t_train, "eval_images_per_s": n_ev / t_eval,
           "train_s": t_train, "eval_s": t_eval,
           "e2e": {"value": (n_tr + n_ev) / e2e_s, "unit": "images/s", "api": "train_epoch + batch_counts (host numpy)"},
           "train_errors": int(stats.n_errors),
           "eval_accuracy": float((np.argmax(cev, axis=1) == d5["eval_labels"]).mean()),
           "api_matches_device_run": bool(np.array_equal(w_api, w) and np.array_equal(cev_api, cev))}
    gp = os.path.join(ROOT, "tests", "golden", "c5_reference.npz")
    if os.path.exists(gp):
        g = np.load(gp)
        wr = g["w_after_60000"]
        ge = os.path.join(ROOT, "tests", "golden", "c5_eval_reference.npz")
        ev_all = bool(np.array_equal(cev, np.load(ge)["eval_counts"])) if os.path.exists(ge) else None
        out["parity"] = {"w_rel_err_vs_reference_after_60000": float(np.abs(w - wr).max() / np.abs(wr).max()),
                         "train_counts_identical_frac": float((ctr == g["train_counts"]).all(axis=1).mean()),
                         "eval_counts_first500_identical": bool(np.array_equal(cev[:500], g["eval_counts_500"])),
                         "c5_eval_all10000_counts_equal_reference": ev_all,
                         "reference_cpu_train_s_60000_build_box": float(g["train_seconds"])}
    cb = line.get("train", {}).get("cpu_baseline", {}).get("value")
    ci_ = line.get("cpu_baseline", {}).get("value")
    if cb and ci_:
        est = n_tr / cb + n_ev / ci_
        out["cpu_baseline"] = {"value": (n_tr + n_ev) / est, "unit": "images/s", "cores": "1 (train) / all (eval)",
                               "kind": line.get("cpu_baseline", {}).get("kind", "port"), "sample": "extrapolated from the timed oracle samples above "
                               "(train: 1 core, sequential as the reference; eval: all host cores)"}
    return out


def bench_latency(sd, d, w_fix, bank):
    """BASELINE configs[3] / SURVEY 8(d) config 4: real-time batch-1 latency.
    Each of the 500 preprocessed synthetic canvases goes through the public
    run_presentation (host uint8 image + float64 weights in, int64 counts
    out) at T = 75 ms, dt = 1 ms, timed per call on the host exactly as the
    reference service times inference_ms (service.py:76-78)."""
    import dataclasses
    imgs = d["c4_images"]
    cfg75 = dataclasses.replace(sd.NetworkConfig(), t=0.075)
    for x in imgs[:20]:
        sd.run_presentation(x, w_fix, bank, cfg75)
    ms = []
    for x in imgs:
        t0 = time.perf_counter()
        sd.run_presentation(x, w_fix, bank, cfg75)
        ms.append((time.perf_counter() - t0) * 1e3)
    ms = np.array(ms)
    gold = np.load(os.path.join(ROOT, "tests", "golden", "c3_counts_reference.npz"))["c4_counts_t75"]
    same = all(np.array_equal(sd.run_presentation(imgs[i], w_fix, bank, cfg75), gold[i]) for i in range(len(gold)))
    return {"metric": "batch-1 run_presentation latency, T=75 ms, dt=1 ms (500 synthetic canvases)",
            "p50_ms": float(np.percentile(ms, 50)), "p99_ms": float(np.percentile(ms, 99)),
            "mean_ms": float(ms.mean()), "max_ms": float(ms.max()), "budget_ms": 100.0,
            "api": "run_presentation (host image + host float64 weights each call)",
            "c4_all500_counts_equal_reference": bool(same)}


def bench_preprocess(sd, w_fix, bank):
    """SURVEY 8(f) GPU preprocess: the 500 synthetic user canvases of config 4
    (tests/golden/canvases.npz, shapes 75-110 px) through preprocess_batch
    (host canvases in, 28x28 images out, one launch) and, per canvas, the
    serving path preprocess_pipeline + run_presentation (T = 75 ms) as
    service.py:146-157 runs it.  Checked against the reference's outputs.
    CPU baseline: the reference's own pipeline with Pillow's C resize
    (oracle.preprocess_oracle.preprocess_pil), one core."""
    import dataclasses
    from oracle import preprocess_oracle as po
    z = np.load(os.path.join(ROOT, "tests", "golden", "canvases.npz"))
    canv = [z["pixels"][o:o + h * w].reshape(h, w) for (h, w), o in zip(z["shapes"][:500], z["offsets"][:500])]
    want = z["outputs"][:500]
    for _ in range(3):
        imgs, blank = sd.preprocess_batch(canv)
    ts = []
    for _ in range(10):
        t0 = time.perf_counter()
        imgs, blank = sd.preprocess_batch(canv)
        ts.append(time.perf_counter() - t0)
    batch_s = statistics.median(ts)
    cfg75 = dataclasses.replace(sd.NetworkConfig(), t=0.075)
    for c in canv[:20]:
        sd.run_presentation(sd.preprocess_pipeline(c), w_fix, bank, cfg75)
    pre_ms, serve_ms = [], []
    for c in canv:
        t0 = time.perf_counter()
        im = sd.preprocess_pipeline(c)
        t1 = time.perf_counter()
        sd.run_presentation(im, w_fix, bank, cfg75)
        t2 = time.perf_counter()
        pre_ms.append((t1 - t0) * 1e3)
        serve_ms.append((t2 - t0) * 1e3)
    k = 200
    t0 = time.perf_counter()
    for c in canv[:k]:
        po.preprocess_pil(c)
    cpu = k / (time.perf_counter() - t0)
    return {"metric": "canvas preprocessing (500 synthetic user canvases -> 28x28), canvases/s", "value": 500 / batch_s,
            "unit": "canvases/s", "api": "preprocess_batch (host canvases in, images out)",
            "batch1_preprocess_p50_ms": float(np.percentile(pre_ms, 50)),
            "serve_p50_ms": float(np.percentile(serve_ms, 50)), "serve_p99_ms": float(np.percentile(serve_ms, 99)),
            "serve_api": "preprocess_pipeline + run_presentation, T=75 ms (service.py:146-157)",
            "outputs_equal_reference": bool(np.array_equal(imgs, want) and not blank.any()),
            "cpu_baseline": {"value": cpu, "unit": "canvases/s", "cores": 1, "kind": "port",
                             "sample": f"first {k} canvases, the reference pipeline with Pillow's C resize "
                                       "(oracle.preprocess_oracle.preprocess_pil)"}}


def cpu_baseline(d, w):
    cores = host_cores()
    imgs = d["c3_images"]
    sample = int(min(len(imgs), max(2 * cores, cores * 64)))   # ~25 core-seconds of CPU work
    fn, kind, desc = reference_infer(imgs, w, cores)
    fn(imgs[: 2 * cores])  # fork + table warm-up
    t0 = time.perf_counter()
    fn(imgs[:sample])
    v = sample / (time.perf_counter() - t0)
    return {"value": v, "unit": "images/s", "cores": cores, "kind": kind,
            "sample": f"first {sample} of the 10,000 c3 images, {desc}, {cpu_model()}"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=int(os.environ.get("WORLD_SIZE", "1")))
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--skip-train", action="store_true")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--skip-latency", action="store_true")
    ap.add_argument("--skip-c5", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
