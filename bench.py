#!/usr/bin/env python
"""Benchmark: H-CNN hash-conv layer forward+backward on synthetic voxelised shells.

A step = one 3x3x3 stride-1 hash-conv layer fwd+bwd over this rank's batch of
whole shapes (`--shapes-per-gpu` copies of the sphere shell of bench.cpp:33-77 at
`--res`), i.e. forward (field probes + gather + contraction), dW, and the input
gradient; with N GPUs each rank runs its own shapes (weak scaling) and dW is
all-reduced over NCCL. The metric is occupied voxels per second (whole job);
shapes/s is reported beside it.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Timing: W untimed warm-up steps, then K steps between barrier+synchronize,
CUDA events on the launching stream, max over ranks. The working set (column
matrices / feature maps of ~1.8M voxels) is far larger than L2, so no flush is
needed. --impl reference runs the unmodified reference CPU library
(oracle/_ref/libhcref.so, built from /root/reference) on rank 0 over a bounded
sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
CACHE = os.path.join(ROOT, "paper_1803_11385_b200", "_cache")
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--res", type=int, default=256)
    p.add_argument("--shapes-per-gpu", type=int, default=8)
    p.add_argument("--cin", type=int, default=64)
    p.add_argument("--cout", type=int, default=64)
    p.add_argument("--path", default="fused", choices=["materialized", "fused"])
    p.add_argument("--dtype", default="f32", choices=["f32", "bf16"],
                   help="fused path: f32 = fp32 operands carried as bf16 hi/lo planes (the reference's fp32 "
                        "within 1e-5, the headline); bf16 = bf16 operands (faster, bf16 tolerance)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-ref-kernels", action="store_true",
                   help="skip the reference-layout operator timings (hash2col/col2hash/pool/unpool vs HBM)")
    p.add_argument("--workload", default="conv", choices=["conv", "net", "seg"],
                   help="conv: one hash-conv layer fwd+bwd (the BASELINE metric); net: a full H-CNN "
                        "classification train step (BASELINE configs 2/3)")
    p.add_argument("--classes", type=int, default=40)
    p.add_argument("--no-graph", action="store_true", help="net workload: time the eager step")
    p.add_argument("--sync-bn", action="store_true",
                   help="net workload, N>1: batch-norm statistics over the global batch (3 small all-reduces per "
                        "BN layer); default: per-rank statistics")
    return p.parse_args()


# ------------------------------------------------------------------ inputs
def shell_levels(res: int):
    """Finest and next-coarser PSH level of the synthetic shell, cached as .psh."""
    from paper_1803_11385_b200.psh import PshLevel, VoxelSet, mix_seed, read_psh_file, write_psh_file
    os.makedirs(CACHE, exist_ok=True)
    path = os.path.join(CACHE, f"shell{res}_l01.psh")
    if os.path.exists(path):
        lv = read_psh_file(path)
        if len(lv) == 2 and lv[0].resolution == res:
            return lv
    s = VoxelSet.sphere(res, True)
    lv = [PshLevel.build(s, mix_seed(1, 0)), PshLevel.build(s.coarsen(), mix_seed(1, 1))]
    tmp = f"{path}.tmp{os.getpid()}"  # ranks of a multi-GPU launch may race to build the cache
    write_psh_file(tmp, lv)
    os.replace(tmp, path)
    return lv


def _device(local: int):
    """One process per GPU (LOCAL_RANK). HCB_TEST_SHARE_GPU=1 folds ranks onto the visible GPUs
    (N>1 code-path checks on a 1-GPU box, with HCB_TEST_DIST_BACKEND=gloo; timings meaningless)."""
    import torch
    if os.environ.get("HCB_TEST_SHARE_GPU") == "1":
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    return torch.device("cuda", local)


def _init_dist(dev):
    import torch.distributed as dist
    backend = os.environ.get("HCB_TEST_DIST_BACKEND", "nccl")
    if backend == "nccl":
        # NCCL's init lines (communicator size, NVLS / NVLink transport) land on stderr
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=dev)
    else:
        dist.init_process_group(backend)
    if dist.get_rank() == 0:
        print(f"[bench] process group: backend={dist.get_backend()} world_size={dist.get_world_size()}",
              file=sys.stderr)


def peaks():
    try:
        with open(PEAKS_PATH) as f:
            return json.load(f), "measured"
    except Exception:
        return FALLBACK_PEAKS, "fallback"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled DURING the timed region.

    NVML (nvidia_ml_py) is polled every ~2 ms from a thread, so even a ~20 ms timed region
    gets several samples; `region(True/False)` brackets the timed region and summary()
    reports the samples taken inside it (all samples if none landed there). Falls back to
    `nvidia-smi -lms 50` when NVML is unavailable."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int):
        self.index, self.proc, self.samples, self.in_region = index, None, [], False
        self.stop = threading.Event()
        self.nvml = None

    def region(self, on: bool):
        self.in_region = on

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            bits = {"hw_slowdown": pynvml.nvmlClocksEventReasonHwSlowdown,
                    "hw_thermal_slowdown": pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": pynvml.nvmlClocksEventReasonSwThermalSlowdown,
                    "sw_power_cap": pynvml.nvmlClocksEventReasonSwPowerCap}
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            self.nvml = pynvml

            def poll():
                while not self.stop.is_set():
                    try:
                        sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                        r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.samples.append((self.in_region, float(sm), float(mx),
                                             {n for n, bit in bits.items() if r & bit}))
                    except Exception:
                        pass
                    time.sleep(0.002)

            self.t = threading.Thread(target=poll, daemon=True)
            self.t.start()
            return self
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm, mx = float(parts[0]), float(parts[1])
            except ValueError:
                continue
            self.samples.append((self.in_region, sm, mx,
                                 {n for n, v in zip(self.NAMES, parts[2:6]) if v.lower() == "active"}))

    def __exit__(self, *a):
        self.stop.set()
        if self.nvml is not None:
            self.t.join(timeout=1)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        inside = [x for x in self.samples if x[0]]
        use = inside or self.samples
        if not use:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        reasons = set().union(*(x[3] for x in use))
        return {"sm_mhz": statistics.median(x[1] for x in use), "sm_max_mhz": max(x[2] for x in use),
                "reasons": sorted(reasons), "samples": len(use), "samples_in_timed_region": len(inside),
                "source": "nvml" if self.nvml is not None else "nvidia-smi"}


# ------------------------------------------------------------------ CPU reference
def _level_arrays(level):
    h, o, t, d = level.arrays()

    class A:
        pass

    a = A()
    a.dim, a.resolution, a.batch = level.dim, level.resolution, 1
    a.hash, a.offsets, a.tags = h, o, t
    a.model_of_slot = np.ones(h.size, np.int32)
    a.hash_acc = np.array([0, h.size], np.int64)
    a.offset_acc = np.array([0, level.offset_cells()], np.int64)
    a.data_acc = np.array([0, level.n], np.int64)
    a.hash_dims = np.array([level.hash_dim], np.int32)
    a.offset_dims = np.array([level.offset_dim], np.int32)
    a.data = d
    a.total_columns = lambda: level.n
    a.total_slots = lambda: h.size
    return a


def _all_host_threads(ref):
    """The reference's OpenMP loops run with every host thread this process may use: torchrun
    exports OMP_NUM_THREADS=1 to each rank, which would leave the reference single-threaded at N>1
    (threading.cpp:24-33 set_thread_override wins over the OpenMP default)."""
    try:
        n = len(os.sched_getaffinity(0))
    except AttributeError:
        n = os.cpu_count() or 1
    ref.lib.hcref_set_threads(int(n))


def cpu_conv_sample(res, cin, cout, reps=1):
    """Time the reference CPU conv layer fwd+bwd (hash2col, matmul, conv_backward —
    cnn_ops.cpp:123-232) on ONE shape of the workload."""
    from oracle.oracle import Ref, Restated, have_ref
    lv = shell_levels(res)
    arr = _level_arrays(lv[0])
    n = lv[0].n
    rng = np.random.default_rng(3)
    x = rng.uniform(-1, 1, (cin, n)).astype(np.float32)
    w = rng.uniform(-1, 1, (cout, cin * 27)).astype(np.float32)
    dy = rng.uniform(-1, 1, (cout, n)).astype(np.float32)
    spec = (3, 1, 0, cin, cout)
    if have_ref():
        ref = Ref()
        _all_host_threads(ref)
        s = ref.super_from(arr)
        kind, cores = "reference", ref.max_threads()

        def run():
            cols = ref.hash2col(s, x, s, spec)
            ref.matmul(w, cols)
            ref.conv_backward(dy, w, cols, s, s, spec)
    else:
        R = Restated()
        kind, cores = "port", 1

        def run():
            cols = R.hash2col(arr, x, arr, spec)
            R.matmul(w, cols)
            R.conv_backward(dy, w, cols, arr, arr, spec)
    best = float("inf")
    for _ in range(reps):
        t0 = time.perf_counter()
        run()
        best = min(best, time.perf_counter() - t0)
    sample = f"1 of the workload's shapes ({res}^3 shell, {n} voxels), conv {cin}->{cout} fwd+bwd, best of {reps}"
    return best, n, kind, cores, sample


# ------------------------------------------------------------------ GPU steps
class MaterializedStep:
    """Reference-layout path through the C ABI: hash2col -> W*cols -> dW = dY*cols^T ->
    dcols = W^T*dY -> col2hash (HC_MATH_FAST contraction)."""

    name = "materialized (reference layout, fp32)"
    dtype = "f32"

    def __init__(self, fine, cin, cout, dev):
        import torch
        from paper_1803_11385_b200 import ops
        self.ops, self.torch = ops, torch
        self.fine = fine
        self.spec = ops.ConvSpec(3, 1, 0, cin, cout)
        N = fine.total_columns()
        g = torch.Generator(device=dev).manual_seed(0)
        self.x = torch.rand((cin, N), device=dev, generator=g) * 2 - 1
        self.w = torch.rand((cout, cin * 27), device=dev, generator=g) * 2 - 1
        self.dy = torch.rand((cout, N), device=dev, generator=g) * 2 - 1
        self.N, self.cin, self.cout = N, cin, cout
        self.x_ref, self.dy_ref = self.x, self.dy
        self.op_names = ["hash2col", "fwd_gemm", "dW_gemm", "dcols_gemm", "col2hash"]

    def run_ref(self, x, w, dy, on_dw=None):
        """Reference-layout device inputs -> reference-layout outputs (y, dw, dx)."""
        return self.run(x, w, dy, None, on_dw)

    def run(self, x, w, dy, marks=None, on_dw=None):
        ops, f, sp = self.ops, self.fine, self.spec
        mark = (lambda i: marks[i].record()) if marks else (lambda i: None)
        with ops.math_mode("fast"):
            mark(0)
            cols = ops.hash2col(f, x, f, sp)
            mark(1)
            y = ops.matmul(w, cols)
            mark(2)
            dw = ops.matmul_trans_b(dy, cols)
            if on_dw:
                on_dw(dw)
            mark(3)
            dcols = ops.matmul_trans_a(w, dy)
            mark(4)
            dx = ops.col2hash(dcols, f, f, sp)
            mark(5)
        return y, dw, dx

    def op_model(self, M, R):
        """Algorithmic bytes / flops per op."""
        s, N, ci, co = 4, self.N, self.cin, self.cout
        gather = 28 * ci * N * s + 10 * M + 3 * R + 16 * N
        # the fp32 contractions over the materialised column matrix (27*ci x N) are bound by
        # moving that matrix (AI = 2*co/(4*(1 + co/(27 ci))) ~ 30 flop/B at 64->64, far below
        # the tensor ridge): algorithmic bytes = column matrix + the C x N operand
        colm = 27 * ci * N * s
        return {"hash2col": ("hbm", gather), "fwd_gemm": ("hbm", colm + co * N * s),
                "dW_gemm": ("hbm", colm + co * N * s), "dcols_gemm": ("hbm", colm + co * N * s),
                "col2hash": ("hbm", gather)}



def _tile(c: int) -> int:
    return next(t for t in (16, 32, 64, 128, 256) if c <= t)


def _padded_operands(torch, conv, cin, cout, N, dev, g):
    """Random reference-layout X (cin x N), W (cout x cin*27), dY (cout x N) — zero-padded to
    the tensor-core channel tile set {16, 32, 64, 128, 256} when cin / cout are not in it (the
    native layer's own padding, conv.HashConv): padded rows and weights are zero, so the real
    channels' results are unchanged; the kernels then run (and are timed) at the padded sizes."""
    cin_p, cout_p = conv._tile_channels(cin), conv._tile_channels(cout)
    x = torch.rand((cin, N), device=dev, generator=g) * 2 - 1
    w = torch.rand((cout, cin * 27), device=dev, generator=g) * 2 - 1
    dy = torch.rand((cout, N), device=dev, generator=g) * 2 - 1
    if (cin_p, cout_p) == (cin, cout):
        return x, w, dy, cin, cout
    xp = torch.zeros((cin_p, N), device=dev)
    xp[:cin] = x
    wp = torch.zeros((cout_p, cin_p * 27), device=dev)
    wp.view(cout_p, cin_p, 27)[:cout, :cin] = w.view(cout, cin, 27)
    dyp = torch.zeros((cout_p, N), device=dev)
    dyp[:cout] = dy
    return xp, wp, dyp, cin_p, cout_p


class FusedStepF32:
    """Native path at the reference's precision (include/hashconv_b200_native.h, split
    precision): field map K0 -> fp32 X and dY split into bf16 hi/lo planes -> tcgen05
    gather-GEMM forward (hi.hi + hi.lo + lo.hi) -> split-K tcgen05 dW (three plane products,
    8192-voxel accumulation chains, fixed-order reduction) -> tcgen05 dX (flipped kernel).
    fp32 in, fp32 out, within 1e-5 (normwise) of the float64 instantiation on unquantised
    inputs (tests/test_conv_f32.py). The column matrix never exists in HBM; weights are
    re-packed every step (they change every optimiser step)."""

    name = "fused implicit-GEMM, fp32 via bf16 hi/lo split (tcgen05, fp32 accumulate)"
    dtype = "f32"
    products = {"fwd_conv": 3, "dW_conv": 3, "dX_conv": 3}  # dW: tri mode (c_out >= 32)

    def __init__(self, fine, cin, cout, dev):
        import torch
        from paper_1803_11385_b200 import conv, ops
        self.ops, self.conv, self.torch = ops, conv, torch
        self.fine = fine
        N = fine.total_columns()
        g = torch.Generator(device=dev).manual_seed(0)
        # reference-layout (channel-major fp32) host-facing tensors (tile-set padded) ...
        self.x_ref, self.w, self.dy_ref, cin_p, cout_p = _padded_operands(torch, conv, cin, cout, N, dev, g)
        self.spec = ops.ConvSpec(3, 1, 0, cin_p, cout_p)
        # ... and the native voxel-major fp32 tensors the layer consumes
        self.x = self.x_ref.t().contiguous()
        self.dy = self.dy_ref.t().contiguous()
        self.ws = conv.DwWorkspace()
        self.N, self.cin, self.cout = N, cin, cout
        self.products = dict(self.products, dW_conv=3 if cout_p >= 32 else 4)  # conv_tc.cu dw_plan: tri mode
        self.op_names = ["field_map", "split_pack", "fwd_conv", "dW_conv", "dX_conv"]

    def _layer(self, fmap, xs, dys, w, marks, on_dw=None):
        conv, sp = self.conv, self.spec
        mark = (lambda i: marks[i].record()) if marks else (lambda i: None)
        wf, wb = conv.pack_weights_x2_fb(w, sp.out_channels, sp.in_channels, 27)  # one launch
        mark(2)
        y = conv.gather_gemm_x2(fmap, xs, wf, sp.out_channels)
        mark(3)
        dw = conv.conv_dw_x2(fmap, xs, dys, self.ws)
        if on_dw:
            on_dw(dw)  # the dW all-reduce overlaps the input gradient below
        mark(4)
        dx = conv.gather_gemm_x2(fmap, dys, wb, sp.in_channels)
        mark(5)
        return y, dw, dx

    def run(self, x, w, dy, marks=None, on_dw=None):
        conv, f, sp = self.conv, self.fine, self.spec
        mark = (lambda i: marks[i].record()) if marks else (lambda i: None)
        mark(0)
        fmap = conv.field_map_native(f, f, sp, conv.TILED)
        mark(1)
        return self._layer(fmap, conv.split(x), conv.split(dy), w, marks, on_dw)

    def run_ref(self, x, w, dy, on_dw=None):
        """The drop-in contract: reference-layout (C x N fp32) device inputs; the boundary
        transpose is fused into the hi/lo split; outputs back in the reference layout."""
        conv, f, sp = self.conv, self.fine, self.spec
        fmap = conv.field_map_native(f, f, sp, conv.TILED)
        y, dw, dx = self._layer(fmap, conv.split(x, channel_major=True), conv.split(dy, channel_major=True), w, None,
                                on_dw)
        return conv.to_channel_major(y), dw, conv.to_channel_major(dx)

    def op_model(self, M, R):
        N, ci, co = self.N, self.cin, self.cout
        fl = 2.0 * co * 27 * ci * N
        kmap = 27 * N * 4 + 10 * M + 3 * R + 16 * N
        # split: read X and dY fp32, write their hi/lo bf16 rows (same bytes); pack: W read twice
        split = 2 * (ci + co) * N * 4 + 2 * co * ci * 27 * 4 * 2
        return {"field_map": ("hbm", kmap), "split_pack": ("hbm", split),
                "fwd_conv": ("flop", fl, (ci + co) * N * 4), "dW_conv": ("flop", fl, (ci + co) * N * 4),
                "dX_conv": ("flop", fl, (ci + co) * N * 4)}


class FusedStep:
    """Native path (include/hashconv_b200_native.h): field map K0 -> tcgen05 gather-GEMM
    forward -> split-K tcgen05 dW -> tcgen05 dX (flipped kernel), bf16 operands, fp32
    accumulation; the column matrix never exists in HBM. Weights are re-packed each step
    (they change every optimiser step)."""

    name = "fused implicit-GEMM (tcgen05, bf16 operands, fp32 accumulate)"
    dtype = "bf16"
    products = {"fwd_conv": 1, "dW_conv": 1, "dX_conv": 1}

    def __init__(self, fine, cin, cout, dev):
        import torch
        from paper_1803_11385_b200 import conv, ops
        self.ops, self.conv, self.torch = ops, conv, torch
        self.fine = fine
        N = fine.total_columns()
        g = torch.Generator(device=dev).manual_seed(0)
        # reference-layout (channel-major fp32) host-facing tensors (tile-set padded) ...
        self.x_ref, self.w, self.dy_ref, cin_p, cout_p = _padded_operands(torch, conv, cin, cout, N, dev, g)
        self.spec = ops.ConvSpec(3, 1, 0, cin_p, cout_p)
        # ... and the native voxel-major bf16 operands the layer consumes
        self.x = conv.to_voxel_major(self.x_ref)
        self.dy = conv.to_voxel_major(self.dy_ref)
        self.ws = conv.DwWorkspace()
        self.N, self.cin, self.cout = N, cin, cout
        self.op_names = ["field_map", "pack_w", "fwd_conv", "dW_conv", "dX_conv"]

    def run(self, x, w, dy, marks=None, on_dw=None):
        ops, conv, f, sp = self.ops, self.conv, self.fine, self.spec
        mark = (lambda i: marks[i].record()) if marks else (lambda i: None)
        bf = self.torch.bfloat16
        mark(0)
        fmap = conv.field_map_native(f, f, sp, conv.TILED)
        mark(1)
        wf = conv.pack_weights(w, sp.out_channels, sp.in_channels, 27, False)
        wb = conv.pack_weights(w, sp.out_channels, sp.in_channels, 27, True)
        mark(2)
        y = conv.gather_gemm(fmap, x, wf, sp.out_channels, bf)
        mark(3)
        dw = conv.conv_dw(fmap, x, dy, self.ws)
        if on_dw:
            on_dw(dw)
        mark(4)
        dx = conv.gather_gemm(fmap, dy, wb, sp.in_channels, bf)
        mark(5)
        return y, dw, dx

    def run_ref(self, x, w, dy, on_dw=None):
        """The drop-in contract: reference-layout (C x N fp32) device inputs, layout change
        at the boundary, the fused layer, results back in the reference layout."""
        conv = self.conv
        y, dw, dx = self.run(conv.to_voxel_major(x), w, conv.to_voxel_major(dy), None, on_dw)
        return conv.to_channel_major(y), dw, conv.to_channel_major(dx)

    def op_model(self, M, R):
        N, ci, co = self.N, self.cin, self.cout
        fl = 2.0 * co * 27 * ci * N
        kmap = 27 * N * 4 + 10 * M + 3 * R + 16 * N
        return {"field_map": ("hbm", kmap), "pack_w": ("hbm", 2 * co * ci * 27 * 6),
                "fwd_conv": ("flop", fl, (ci + co) * N * 2), "dW_conv": ("flop", fl, (ci + co) * N * 2),
                "dX_conv": ("flop", fl, (ci + co) * N * 2)}

    def smem_model(self):
        """Shared-memory bytes per launch of the fused kernels (the binding unit at C <= 64,
        DESIGN.md): every 128-row x 64-K stage writes its gathered A tile (cp.async) and B tile
        (TMA) and the SS-form MMA reads both back. dW: per 64-voxel stage each m-tile writes and
        reads a 16 KB gathered tile and reads the group's dY tile (written once per group)."""
        N, ci, co = self.N, self.cin, self.cout
        tiles = (N + 127) // 128
        kst = 27 * ((ci + 63) // 64)  # K stages per forward tile (per dX tile with ci <-> co)
        fwd = tiles * kst * 2 * (128 * 128 + co * 128)
        dx = tiles * 27 * ((co + 63) // 64) * 2 * (128 * 128 + ci * 128)
        mt = (27 * ci + 127) // 128  # dW m-tiles, grouped <= 4 per CTA
        groups = (mt + 3) // 4
        dw = ((N + 63) // 64) * (mt * (2 * 128 * 128 + co * 128) + groups * co * 128)
        return {"fwd_conv": fwd, "dX_conv": dx, "dW_conv": dw}


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.workload == "net":
        return net_main(args, rank, world, local)
    if args.workload == "seg":
        return seg_main(args, rank, world, local)
    if args.impl == "reference":
        return reference_arm(args, rank, world)

    import torch
    import torch.distributed as dist
    dev = _device(local)
    if world > 1:
        _init_dist(dev)

    from paper_1803_11385_b200 import _lib
    from paper_1803_11385_b200.psh import SuperPsh

    from paper_1803_11385_b200.dist import local_levels
    lv = shell_levels(args.res)
    # global batch of shapes_per_gpu * world shells; this rank owns a contiguous block
    fine = SuperPsh.from_levels(local_levels([lv[0]] * (args.shapes_per_gpu * world), world, rank))
    if args.path == "fused":
        step = (FusedStepF32 if args.dtype == "f32" else FusedStep)(fine, args.cin, args.cout, dev)
    else:
        step = MaterializedStep(fine, args.cin, args.cout, dev)
    N = fine.total_columns()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # The one data-path exchange: dW summed over ranks. It is launched on a side
    # stream as soon as the dW kernel is enqueued, so the collective overlaps the input gradient;
    # the step ends when both are done.
    side = torch.cuda.Stream() if world > 1 else None
    pending = []

    def on_dw(dw):
        if world > 1:
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                pending.append(dist.all_reduce(dw, op=dist.ReduceOp.SUM, async_op=True))

    def finish():
        while pending:
            pending.pop().wait()  # the current stream waits for the collective

    def one(marks=None):
        y, dw, dx = step.run(step.x, step.w, step.dy, marks, on_dw)
        finish()
        return dx

    args.warmup = max(args.warmup, 3)
    nops = len(step.op_names)
    per_op = [0.0] * nops
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    marks_all = [[torch.cuda.Event(enable_timing=True) for _ in range(nops + 1)] for _ in range(args.steps)]
    with ClockSampler(local) as clk:  # sampling spans warm-up and the timed region
        for _ in range(args.warmup):
            one()
        barrier()
        launches0 = _lib.lib.hc_launch_count()
        barrier()
        clk.region(True)
        start.record()
        for k in range(args.steps):
            one(marks_all[k])
        end.record()
        barrier()
        clk.region(False)
        launches = _lib.lib.hc_launch_count() - launches0
    elapsed_ms = start.elapsed_time(end)
    for m in marks_all:
        for i in range(nops):
            per_op[i] += m[i].elapsed_time(m[i + 1])
    t = torch.tensor([elapsed_ms], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = float(t.item()) / args.steps
    total_vox = N * world
    value = total_vox / (ms_step / 1e3)

    # ---- e2e through the public API with host buffers (H2D inputs, D2H results)
    e2e = None
    if not args.no_e2e:
        hx = step.x_ref.cpu().pin_memory()
        hw = step.w.cpu().pin_memory()
        hdy = step.dy_ref.cpu().pin_memory()
        cin_p, cout_p = step.spec.in_channels, step.spec.out_channels  # = cin / cout unless tile-padded
        outs = [torch.empty((cout_p, N), pin_memory=True), torch.empty((cout_p, cin_p * 27), pin_memory=True),
                torch.empty((cin_p, N), pin_memory=True)]

        # Pipelined across steps: H2D of step k+1 and D2H of step k-1 run on their own
        # copy streams (independent copy engines) while step k computes; NSLOT slots of
        # device staging buffers; every byte of every step still crosses PCIe.
        comp = torch.cuda.current_stream()
        h2d_s, d2h_s = torch.cuda.Stream(), torch.cuda.Stream()
        NSLOT = int(os.environ.get("HCB_E2E_SLOTS", "3"))  # 3 decouples H2D(k+1) from compute(k-1)
        slots = [dict(x=torch.empty_like(step.x_ref), w=torch.empty_like(step.w), dy=torch.empty_like(step.dy_ref),
                      out=[torch.empty_like(o).pin_memory() for o in outs], free=torch.cuda.Event(),
                      ready=torch.cuda.Event(), done=torch.cuda.Event()) for _ in range(NSLOT)]
        for sl in slots:
            sl["free"].record(comp)

        def e2e_step(k):
            sl = slots[k % NSLOT]
            h2d_s.wait_event(sl["free"])
            with torch.cuda.stream(h2d_s):
                sl["x"].copy_(hx, non_blocking=True)
                sl["w"].copy_(hw, non_blocking=True)
                sl["dy"].copy_(hdy, non_blocking=True)
                sl["ready"].record(h2d_s)
            comp.wait_event(sl["ready"])
            y, dw, dx = step.run_ref(sl["x"], sl["w"], sl["dy"], on_dw)
            sl["free"].record(comp)
            finish()
            sl["done"].record(comp)
            d2h_s.wait_event(sl["done"])
            with torch.cuda.stream(d2h_s):
                for o, r in zip(sl["out"], (y, dw, dx)):
                    r.record_stream(d2h_s)
                    o.copy_(r, non_blocking=True)

        e2e_step(0)
        comp.wait_stream(d2h_s)
        barrier()
        es, ee = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ke = max(50, args.steps)  # long enough that pipeline fill / drain amortise (~1 step of 50)
        es.record(comp)
        for k in range(ke):
            e2e_step(k)
        comp.wait_stream(d2h_s)  # the last results are on the host inside the timed region
        ee.record(comp)
        barrier()
        et = torch.tensor([es.elapsed_time(ee) / ke], device=dev)
        if world > 1:
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
        h2d = (hx.numel() + hw.numel() + hdy.numel()) * 4
        d2h = sum(o.numel() for o in outs) * 4
        e2e = {"value": total_vox / (float(et.item()) / 1e3), "unit": "voxels/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": float(et.item())}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel. Denominators (MEASURED_PEAKS.json): the burst bf16
    # figure for a timed region short enough to run at max clock (this one: ms at ~1965 MHz),
    # the sustained one when the sampled SM clock sat below max (power-capped long runs).
    pk, pk_kind = peaks()
    cs = clk.summary()
    at_max = bool(cs.get("sm_mhz") and cs.get("sm_max_mhz") and cs["sm_mhz"] >= 0.95 * cs["sm_max_mhz"])
    tc_peak = pk["bf16_tflops"] if at_max else pk["bf16_tflops_sustained"]
    tc_basis = "bf16_tflops (burst: timed region at max SM clock)" if at_max else \
        "bf16_tflops_sustained (SM clock below max during the timed region)"
    info = np.zeros(6, np.int64)
    import ctypes
    _lib.lib.hc_psh_info(fine._h, info.ctypes.data_as(ctypes.c_void_p))
    model = step.op_model(int(info[3]), int(info[4]))
    kernels = {}
    for i, name in enumerate(step.op_names):
        avg_ms = per_op[i] / args.steps
        kind, amount = model[name][:2]
        if kind == "hbm":
            ach = amount / (avg_ms / 1e3) / 1e9
            kernels[name] = {"ms": avg_ms, "bound": "hbm", "achieved_GBps": ach,
                             "frac": ach / pk["hbm_gbs"], "algorithmic_bytes": amount}
        else:
            # achieved = the reference's algorithmic flops (2*Cout*27*Cin*N) per second; the
            # split-precision kernels execute `products` bf16 MMAs per fp32 MAC, so their
            # tensor-pipe ceiling is the bf16 peak / products
            ach = amount / (avg_ms / 1e3) / 1e12
            prod = getattr(step, "products", {}).get(name, 1)
            kernels[name] = {"ms": avg_ms, "achieved_TFLOPs": ach, "flops": amount, "bf16_products": prod,
                             "peak_TFLOPs": tc_peak / prod, "frac_tensor": ach * prod / tc_peak}
            if len(model[name]) > 2:
                kernels[name]["algorithmic_bytes"] = model[name][2]
                kernels[name]["arith_intensity"] = amount / model[name][2]
    if hasattr(step, "smem_model"):  # shared-memory traffic per SM-clock (clock sampled in the run)
        clk_mhz = clk.summary().get("sm_mhz") or 1965.0
        for name, nbytes in step.smem_model().items():
            if name in kernels:
                per_clk = nbytes / (kernels[name]["ms"] / 1e3) / (pk.get("sms", 148) * clk_mhz * 1e6)
                kernels[name]["smem_bytes"] = nbytes
                kernels[name]["smem_B_per_clk_per_sm"] = per_clk  # fills + MMA operand reads (traffic figure)
    kpath = os.path.join(ROOT, "profiles", "ncu_kernels.json")
    if os.path.exists(kpath):  # ncu counters of the same kernels (one --set full capture, profiles/)
        try:
            ncu_k = json.load(open(kpath))
            for name in kernels:
                src = "fwd_conv" if name == "dX_conv" else name  # dX runs the forward kernel
                if src in ncu_k:
                    kernels[name]["ncu"] = ncu_k[src]
        except Exception:  # noqa: BLE001 — evidence only
            pass
    dom = max(step.op_names, key=lambda n: per_op[step.op_names.index(n)])
    dk = kernels[dom]
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(dom)
        except Exception:
            traffic = None
    if dk.get("bound") == "hbm":
        roof = {"bound": "hbm", "kernel": dom, "achieved": dk["achieved_GBps"], "peak": pk["hbm_gbs"],
                "unit": "GB/s", "frac": dk["frac"], "traffic": traffic, "peak_source": pk_kind}
    else:
        ach = dk["achieved_TFLOPs"]
        peak = dk["peak_TFLOPs"]
        roof = {"bound": "tensor", "kernel": dom, "achieved": ach, "peak": peak, "unit": "TFLOP/s",
                "frac": ach / peak, "traffic": traffic, "peak_source": pk_kind,
                "peak_basis": tc_basis + (f" / {dk['bf16_products']} bf16 products per fp32 MAC"
                                          if dk["bf16_products"] > 1 else "")}

    ref_layout = None
    if not args.no_ref_kernels and args.path == "fused":
        try:
            ref_layout = ref_layout_kernels(args.res, args.shapes_per_gpu, args.cin, pk["hbm_gbs"])
        except Exception as e:  # noqa: BLE001 — reported, never fatal for the headline
            ref_layout = {"error": repr(e)}

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        secs, n1, kind, cores, sample = cpu_conv_sample(args.res, args.cin, args.cout)
        cpu = {"value": n1 / secs, "unit": "voxels/s", "cores": cores, "kind": kind, "sample": sample}

    line = {
        "metric": "hash-conv fwd+bwd occupied voxels/sec",
        "value": value, "unit": "voxels/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": step.dtype, "data": "synthetic (sphere shells, bench.cpp:33-77; uniform[-1,1] features/weights)",
        "config": dict(conv_config(args, world), voxels_per_gpu=N, path=step.name,
                       l2="working set >> L2 (no flush needed)"),
        "shapes_per_s": args.shapes_per_gpu * world / (ms_step / 1e3),
        "roofline": roof, "kernels": kernels, "ref_layout_kernels": ref_layout, "cpu_baseline": cpu, "e2e": e2e,
        "gpu_launches": int(launches), "clocks": cs,
        "comm": {"backend": dist.get_backend() if world > 1 else None, "world_size": world,
                 "collective": "one all_reduce(sum) of dW per step on a side stream, overlapping dX"
                 if world > 1 else None},
    }
    print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def ref_layout_kernels(res, shapes, C, hbm_gbs, reps=5):
    """The reference-layout operators (include/hashconv_b200.h: hash2col, col2hash, max_pool,
    max_unpool, the K0 field map) at the bench workload, fp32 C x N operands, vs the HBM
    roofline. Algorithmic bytes per SURVEY.md §8d: hash2col / col2hash (27+1)*C*N*4 + 10*M +
    3*R + 16*N; max_pool C*Nf*4 + C*Nc*8; max_unpool C*Nc*8 + C*Nf*4; field map 27*N*4 + 10*M +
    3*R + 16*N. CUDA events around `reps` back-to-back calls (operands >> L2)."""
    import torch
    from paper_1803_11385_b200 import ops
    from paper_1803_11385_b200.psh import SuperPsh
    lv = shell_levels(res)
    fine, coarse = SuperPsh.from_levels([lv[0]] * shapes), SuperPsh.from_levels([lv[1]] * shapes)
    N, Nc, M, R = fine.total_columns(), coarse.total_columns(), fine.M, fine.R
    sp, pool = ops.ConvSpec(3, 1, 0, C, C), ops.ConvSpec(2, 2, 0, C, C)
    g = torch.Generator(device="cuda").manual_seed(9)
    x = torch.rand((C, N), device="cuda", generator=g) * 2 - 1
    cols = ops.hash2col(fine, x, fine, sp)
    mp = ops.max_pool(fine, x, coarse, pool)
    gather = 28 * C * N * 4 + 10 * M + 3 * R + 16 * N
    rows = [("field_map", lambda: ops.field_map(fine, fine, sp), 27 * N * 4 + 10 * M + 3 * R + 16 * N),
            ("hash2col", lambda: ops.hash2col(fine, x, fine, sp), gather),
            ("col2hash", lambda: ops.col2hash(cols, fine, fine, sp), gather),
            ("max_pool", lambda: ops.max_pool(fine, x, coarse, pool), C * N * 4 + C * Nc * 8),
            ("max_unpool", lambda: ops.max_unpool(mp.output, mp.switches, fine, coarse, pool, check_now=False),
             C * Nc * 8 + C * N * 4)]
    out = {}
    for name, fn, nbytes in rows:
        fn()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(reps):
            fn()
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / reps
        gbs = nbytes / (ms / 1e3) / 1e9
        out[name] = {"ms": ms, "algorithmic_bytes": nbytes, "achieved_GBps": gbs, "frac": gbs / hbm_gbs}
    ops.check_deferred()
    del cols
    torch.cuda.empty_cache()
    return {"workload": f"{res}^3 shell x {shapes}, C={C} fp32 (reference layout C x N)", "N_fine": N,
            "N_coarse": Nc, "peak_GBps": hbm_gbs, "kernels": out}


def conv_config(args, world):
    """The conv workload descriptor, shared by both arms (the reference arm times a bounded
    sample of this same workload)."""
    return {"workload": f"{args.res}^3 shell x {args.shapes_per_gpu}/GPU, 3x3x3 hash-conv "
                        f"{args.cin}->{args.cout} fwd+bwd (BASELINE config 4 per-GPU shard)",
            "res": args.res, "shapes_per_gpu": args.shapes_per_gpu, "global_batch": args.shapes_per_gpu * world,
            "c_in": args.cin, "c_out": args.cout, "parallelism": f"dp{world} (shapes sharded, dW all-reduce)",
            "channels_padded_to": None if (args.cin, args.cout) == (_tile(args.cin), _tile(args.cout))
            else [_tile(args.cin), _tile(args.cout)]}


def reference_arm(args, rank, world):
    """--impl reference: the unmodified reference CPU library on rank 0 only."""
    if rank != 0:
        return
    import ctypes  # noqa: F401
    from oracle.oracle import have_ref
    if not have_ref():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libhcref.so not built"}))
        return
    for _ in range(args.warmup and 1):
        cpu_conv_sample(args.res, args.cin, args.cout)
    times = []
    n1 = None
    kind = cores = sample = None
    for _ in range(args.steps):
        secs, n1, kind, cores, sample = cpu_conv_sample(args.res, args.cin, args.cout)
        times.append(secs)
    ms = 1e3 * sum(times) / len(times)
    value = n1 / (ms / 1e3)
    print(json.dumps({
        "impl": "reference", "metric": "hash-conv fwd+bwd occupied voxels/sec", "value": value, "unit": "voxels/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (sphere shells, bench.cpp:33-77; uniform[-1,1] features/weights)",
        "config": dict(conv_config(args, world), sample_voxels_per_step=n1,
                       sample_note=f"each step times 1 of the workload's {args.shapes_per_gpu} identical shapes "
                               "(the reference's cost is linear in voxels, so voxels/s is the workload's rate)",
                       path="reference CPU (oracle/_ref: the unmodified reference library)"),
        "cpu_baseline": {"value": value, "unit": "voxels/s", "cores": cores, "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": "voxels/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))


# ------------------------------------------------------------------ net workload
def shell_pyramid(res: int):
    """build_pyramid (net.cpp:19-32) of the synthetic shell, cached as .psh."""
    from paper_1803_11385_b200.psh import VoxelSet, build_pyramid, read_psh_file, write_psh_file
    os.makedirs(CACHE, exist_ok=True)
    path = os.path.join(CACHE, f"shell{res}_pyramid.psh")
    if os.path.exists(path):
        lv = read_psh_file(path)
        if lv and lv[0].resolution == res and lv[-1].resolution == 4:
            return lv
    lv = build_pyramid(VoxelSet.sphere(res, True), 1)
    tmp = f"{path}.tmp{os.getpid()}"  # ranks of a multi-GPU launch may race to build the cache
    write_psh_file(tmp, lv)
    os.replace(tmp, path)
    return lv


def cpu_net_sample(res: int, b: int, classes: int):
    """The reference net's net_loss_and_gradients (net.cpp:260-323) on b shell copies."""
    from oracle.oracle import Ref
    ref = Ref()
    _all_host_threads(ref)
    s = ref.sphere_set(res, True)
    levels, cur, i = [], s, 0
    while True:
        levels.append(ref.build_psh(cur, 0))
        if cur.resolution == 4:
            break
        cur = ref.coarsen(cur)
        i += 1
    supers = [ref.build_super([lv] * b) for lv in levels]
    lmax = int(round(np.log2(res)))
    rn = ref.net_make(lmax, classes, 7)
    labels = np.arange(b, dtype=np.int32) % classes
    t0 = time.perf_counter()
    rn.loss_and_gradients(supers, labels, classes, 1024)
    return time.perf_counter() - t0, ref.max_threads()


def net_main(args, rank, world, local):
    """H-CNN classification train step (net.cpp:349-375) on the native path: per-batch maps +
    forward + loss + backward + SGD; b shells per GPU, weight gradients all-reduced."""
    import torch
    import torch.distributed as dist
    if args.impl == "reference":
        if rank != 0:
            return
        b = 2
        secs, cores = cpu_net_sample(args.res, b, args.classes)
        v = b / secs
        print(json.dumps({"impl": "reference", "metric": "hcnn train step shapes/sec", "value": v,
                          "unit": "shapes/s", "n_gpus": world, "steps": 1, "warmup": 0, "ms_per_step": secs * 1e3,
                          "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
                          "data": "synthetic", "config": {"workload": f"hcnn net {args.res}^3 x {b} shells"},
                          "cpu_baseline": {"value": v, "unit": "shapes/s", "cores": cores, "kind": "reference",
                                           "sample": f"{b} shells, loss+gradients"},
                          "e2e": {"value": v, "unit": "shapes/s", "h2d_bytes_per_step": 0,
                                  "d2h_bytes_per_step": 0}}))
        return
    dev = _device(local)
    if world > 1:
        _init_dist(dev)
    from paper_1803_11385_b200 import _lib
    from paper_1803_11385_b200 import net as nnet
    from paper_1803_11385_b200.dist import allreduce_gradients, sum_over_ranks
    from paper_1803_11385_b200.psh import SuperPsh
    pyr = shell_pyramid(args.res)
    b = args.shapes_per_gpu
    lmax = int(round(np.log2(args.res)))
    levels = [SuperPsh.from_levels([lv] * b) for lv in pyr]
    feats = np.concatenate([pyr[0].arrays()[3]] * b, axis=1)
    # every rank starts from the same weights (data parallelism)
    net = nnet.NativeHashNet(lmax, args.classes, seed=0,
                             sync_bn=sum_over_ranks if (args.sync_bn and world > 1) else None, precision=args.dtype)
    x = net.input_features(torch.from_numpy(np.ascontiguousarray(feats)).to(dev))
    labels = torch.randint(0, args.classes, (b,), device=dev)
    voxels = sum(s.total_columns() for s in levels)

    def eager():
        nb = nnet.NetBatch.build(levels)  # the batch's K0 / pool / dense-pool maps: per step
        return net.train_step(nb, x, labels, allreduce_gradients, b * world)

    one = eager
    mode = "eager"
    if not args.no_graph and world == 1:
        try:  # the whole step as one CUDA graph (per-batch maps included in the graph)
            one = nnet.GraphedStep(net, levels, x, labels, allreduce_gradients, b * world)
            mode = "cuda-graph"
        except Exception as e:  # noqa: BLE001 — report and time the eager step instead
            print(f"cuda graph capture failed ({e}); timing the eager step", file=sys.stderr)
            one = eager

    # The small nets' working sets fit in the 126 MB L2: each timed step is bracketed by its
    # own events and preceded (outside the bracket) by a 256 MB write that flushes L2.
    flush = torch.empty(256 * 2 ** 20 // 4, dtype=torch.float32, device=dev)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(local) as clk:  # sampling spans warm-up and the timed region
        for _ in range(max(3, args.warmup)):
            one()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        launches0 = _lib.lib.hc_launch_count()
        clk.region(True)
        for e0, e1 in evs:
            flush.zero_()
            e0.record()
            one()
            e1.record()
        torch.cuda.synchronize()
        clk.region(False)
        launches = _lib.lib.hc_launch_count() - launches0
        if mode == "cuda-graph":  # graph replays bypass the host launch counter
            launches = one.launches_per_step * args.steps
    t = torch.tensor([sum(e0.elapsed_time(e1) for e0, e1 in evs) / args.steps], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            secs, cores = cpu_net_sample(args.res, 2, args.classes)
            cpu = {"value": 2 / secs, "unit": "shapes/s", "cores": cores, "kind": "reference",
                   "sample": "2 shells, net_loss_and_gradients"}
        # the paper's GPU (GTX 1080, Caffe) classification-net iteration at batch 32
        # (Table 2) -> shapes/s; comparable only at that batch
        paper = {32: 1270.0, 64: 438.0, 128: 147.0, 256: 40.3, 512: 12.3}
        value = b * world / (ms / 1e3)
        vs = value / paper[args.res] if (b * world == 32 and args.res in paper) else None
        print(json.dumps({
            "metric": "hcnn train step shapes/sec", "value": value, "unit": "shapes/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": vs,
            "vs_baseline_source": "paper GPU net iteration, batch 32 (BASELINE.md §1, PAPER.md:485)" if vs else None,
            "dtype": args.dtype,
            "precision_note": "f32: fp32 activations, conv fwd/dW/dX via bf16 hi/lo split on tcgen05 (within 1e-5 "
                              "of the fp32 reference net step, tests/test_net_gpu.py)" if args.dtype == "f32" else
                              "bf16 conv operands and activations, fp32 accumulation",
            "data": "synthetic (sphere shell pyramid, bench.cpp:33-77; random labels)",
            "config": {"workload": f"hcnn classification net {args.res}^3, {lmax - 1} conv/pool levels, "
                                   f"{b} shells/GPU", "res": args.res, "global_batch": b * world,
                       "classes": args.classes, "voxels_per_gpu_all_levels": voxels,
                       "parallelism": f"dp{world}", "launch": mode,
                       "l2": "flushed before every timed step (256 MB write outside the step's events)",
                       "batch_norm": "global-batch (sync)" if net.sync_bn is not None else "per-rank"},
            "voxels_per_s": voxels * world / (ms / 1e3), "cpu_baseline": cpu, "gpu_launches": int(launches),
            "clocks": clk.summary()}))
    if world > 1:
        dist.destroy_process_group()


# ------------------------------------------------------------------ segmentation workload
def seg_main(args, rank, world, local):
    """BASELINE config 4's composition: a SegNet/DeconvNet-style encoder-decoder training step
    on the 256^3 shell level pair (conv, BN+ReLU, max pool, conv, unpool + stride-2 deconv,
    conv, per-voxel softmax, SGD), --shapes-per-gpu shells per GPU, C = --cin channels."""
    import torch
    import torch.distributed as dist
    if args.impl == "reference":
        if rank == 0:
            print(json.dumps({"impl": "reference", "unavailable": "the reference has no segmentation net "
                                                                  "(only its operators: see --workload conv)"}))
        return
    dev = _device(local)
    if world > 1:
        _init_dist(dev)
    from paper_1803_11385_b200 import _lib
    from paper_1803_11385_b200.psh import SuperPsh
    from paper_1803_11385_b200.dist import allreduce_gradients
    from paper_1803_11385_b200.seg import NativeSegNet
    lv = shell_levels(args.res)
    b = args.shapes_per_gpu
    fine, coarse = SuperPsh.from_levels([lv[0]] * b), SuperPsh.from_levels([lv[1]] * b)
    seg = NativeSegNet(fine, coarse, c_in=8, c=args.cin, classes=16, seed=rank, precision=args.dtype)
    g = torch.Generator(device=dev).manual_seed(rank)
    nf = fine.total_columns()
    x = torch.rand((nf, 8), device=dev, generator=g) * 2 - 1
    if args.dtype == "bf16":
        x = x.to(torch.bfloat16)
    labels = torch.randint(0, 16, (nf,), device=dev, generator=g)
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        for _ in range(max(3, args.warmup)):
            seg.step(x, labels, allreduce_gradients, world)
        torch.cuda.synchronize()
        launches0 = _lib.lib.hc_launch_count()
        clk.region(True)
        st.record()
        for _ in range(args.steps):
            seg.step(x, labels, allreduce_gradients, world)
        en.record()
        torch.cuda.synchronize()
        clk.region(False)
        launches = _lib.lib.hc_launch_count() - launches0
    t = torch.tensor([st.elapsed_time(en) / args.steps], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    if rank == 0:
        print(json.dumps({
            "metric": "segmentation train step occupied voxels/sec", "value": nf * world / (ms / 1e3),
            "unit": "voxels/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": args.dtype,
            "data": "synthetic (sphere shells; random features and per-voxel labels)",
            "config": {"workload": f"seg encoder-decoder {args.res}^3 -> {args.res // 2}^3 -> {args.res}^3, "
                                   f"{b} shells/GPU, C={args.cin}", "res": args.res, "global_batch": b * world,
                       "fine_voxels_per_gpu": nf, "coarse_voxels_per_gpu": coarse.total_columns(),
                       "parallelism": f"dp{world} (shapes sharded, weight gradients all-reduced)",
                       "l2": "working set >> L2 (activations of 1.8 M fine voxels; no flush needed)"},
            "shapes_per_s": b * world / (ms / 1e3), "gpu_launches": int(launches), "clocks": clk.summary()}))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
