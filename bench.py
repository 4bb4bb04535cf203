#!/usr/bin/env python
"""bench.py -- AG+GEMM & Flash Decode latency on B200 (BASELINE.json metric).

Headline (one JSON line on rank 0): the fused All-Gather+GEMM step of
BASELINE.json configs[1] -- bf16, M=8192 gathered rows, K=8192 (A sharded
along K), N=28672/W per GPU -- timed with CUDA events over K back-to-back
steps after W warm-ups, max over ranks.  Every input is larger than L2
(A 128 MiB, B 448 MiB at W=1), so no flush is needed between steps.

Beside it, in the same line: per-step percentiles (the reference reports
median/p10/p90, proj/tools/bench.cpp:143-144, 351-353), the roofline of the
dominant kernel, the NCCL+cuBLAS BSP baseline, an end-to-end number through
the C ABI with host buffers, NVML clocks (sampled, plus the driver's
power/thermal violation counters over each section), the reference's CPU
path (oracle/_ref, timed on this host), and as `secondary` the Flash Decode
configs (configs[2], configs[3]: fused vs the library's BSP schedule vs an
NCCL BSP arm of attention kernel -> all_gather_into_tensor -> combine
kernel) and the config-5 M sweep, each with its roofline, numerics and CPU
baseline.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
  torchrun --nproc-per-node N bench.py --gpus N ...
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

M_, K_, N_TOTAL = 8192, 8192, 28672
FD3 = dict(batch=1, q_heads=64, kv_heads=8, head_dim=128, kv_len=131072)
FD4 = dict(batch=32, q_heads=64, kv_heads=8, head_dim=128, kv_len=32768)
SWEEP_MS = (128, 256, 512, 1024, 2048, 4096, 8192, 16384)
METRIC = "AG+GEMM & Flash Decode latency (µs) at 1/2/4/8 B200 vs BSP; % of roofline"
# NVLink 5 per GPU and direction: the pool's measured peer copy and the
# nominal figure (/opt/skills/guides/B200_PROFILING.md).
NVLINK_MEASURED_GBS, NVLINK_NOMINAL_GBS = 770.0, 900.0
BF16_OUT_TOL = 2.0 ** -8 + 1e-4  # bf16 output rounding (2^-8 of the head's max) + the fp32-grade path
F32_OUT_TOL = 1e-4


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return dict(hbm=p["hbm_gbs"], bf16=p["bf16_tflops"], bf16_sus=p["bf16_tflops_sustained"],
                    src="measured")
    except Exception:
        return dict(hbm=6650.0, bf16=1590.0, bf16_sus=1400.0, src="fallback")


def ncu_traffic(key):
    """dram bytes per launch of the dominant kernel from the committed
    ncu --set full summary (profiles/ncu_summary.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            return json.load(f).get(key, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


class ClockSampler:
    """Clocks and throttle reasons during a timed section (NVML): SM clock and
    the active event-reason mask sampled every 2 ms, plus the driver's own
    power / thermal violation-time counters read before and after the section
    (they cover the whole section, not just the sample points)."""

    REASONS = {0x2: "applications_clocks", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake",
               0x100: "display_clocks"}

    def __init__(self, dev=0):
        self.samples, self.reasons, self.stop = [], set(), threading.Event()
        self.max_mhz = None
        self.viol0 = self.viol1 = None
        try:
            import pynvml as N
            N.nvmlInit()
            self.N = N
            self.h = N.nvmlDeviceGetHandleByIndex(dev)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
        except Exception:
            self.N = None

    def _violations(self):
        N = self.N
        out = {}
        for name, pol in (("power", "NVML_PERF_POLICY_POWER"), ("thermal", "NVML_PERF_POLICY_THERMAL"),
                          ("board_limit", "NVML_PERF_POLICY_BOARD_LIMIT"),
                          ("reliability", "NVML_PERF_POLICY_RELIABILITY")):
            try:
                out[name] = int(N.nvmlDeviceGetViolationStatus(self.h, getattr(N, pol)).violationTime)
            except Exception:
                pass
        return out

    def _run(self):
        N = self.N
        while not self.stop.is_set():
            try:
                self.samples.append(N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM))
                mask = N.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.N:
            self.viol0 = self._violations()
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        if self.N:
            self.t.join()
            self.viol1 = self._violations()

    def summary(self):
        s = {"sm_mhz": statistics.median(self.samples) if self.samples else None,
             "sm_min_mhz": min(self.samples) if self.samples else None,
             "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}
        if self.viol0 is not None and self.viol1 is not None:
            s["violation_ms"] = {k: round((self.viol1[k] - self.viol0[k]) / 1e6, 3) for k in self.viol1
                                 if k in self.viol0}
        return s


# ---------------------------------------------------------------------------------
# distributed plumbing (torchrun) -- one process per GPU, IPC symmetric heap

def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class Ctx:
    def __init__(self, n_gpus):
        import torch
        self.torch = torch
        self.ws, self.rank, self.local = dist_env()
        if self.ws != n_gpus and self.ws > 1:
            raise SystemExit(f"--gpus {n_gpus} but WORLD_SIZE={self.ws}")
        self.W = max(self.ws, 1)
        # TFB_BENCH_SHARED_GPU=1: every rank on GPU 0 with gloo plumbing -- a
        # test mode that exercises the multi-process (IPC) paths on a one-GPU
        # box; its numbers are not scaling numbers.
        self.shared = os.environ.get("TFB_BENCH_SHARED_GPU") == "1" and self.ws > 1
        if self.shared:
            self.local = 0
        torch.cuda.set_device(self.local)
        self.dev = torch.device("cuda", self.local)
        if self.ws > 1:
            import torch.distributed as dist
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            if self.shared:
                dist.init_process_group("gloo")
            else:
                dist.init_process_group("nccl", device_id=self.dev)
            self.dist = dist

    def all_gather(self, out, inp):
        """all_gather_into_tensor (NCCL, on the current stream); through host
        memory in shared-GPU test mode."""
        if self.W == 1:
            out.copy_(inp.view_as(out))
            return
        if not self.shared:
            self.dist.all_gather_into_tensor(out, inp)
            return
        parts = [self.torch.empty_like(inp, device="cpu") for _ in range(self.ws)]
        self.dist.all_gather(parts, inp.cpu())
        out.copy_(self.torch.stack(parts).view_as(out))

    def barrier(self):
        if self.ws > 1:
            self.dist.barrier()

    def max(self, x: float) -> float:
        if self.ws == 1:
            return x
        from paper_2511_02168_b200.dist import max_over_ranks
        return max_over_ranks(self.dist, x, None if self.shared else self.dev)

    def all_true(self, b: bool) -> bool:
        return self.max(0.0 if b else 1.0) == 0.0

    def world(self, heap_bytes):
        import paper_2511_02168_b200 as tf
        from paper_2511_02168_b200 import _abi
        L = _abi.lib()
        h = C.c_void_p()
        if self.ws == 1:
            devs = (C.c_int * 1)(self.local)
            _abi.check(L.tf_world_create(1, devs, heap_bytes, 0.0, C.byref(h)))
        else:
            _abi.check(L.tf_world_create_ipc(self.rank, self.ws, self.local, heap_bytes, 0.0, C.byref(h)))
            from paper_2511_02168_b200.dist import gather_ipc_handles
            mine = (C.c_char * _abi.IPC_HANDLE_BYTES)()
            _abi.check(L.tf_world_ipc_export(h, mine))
            allh = gather_ipc_handles(self.dist, bytes(mine), self.ws)
            buf = (C.c_char * (_abi.IPC_HANDLE_BYTES * self.ws)).from_buffer_copy(allh)
            _abi.check(L.tf_world_ipc_import(h, buf))
        w = tf.World.__new__(tf.World)
        w.lib, w.W, w.devices, w.handle = L, self.W, [self.local] * self.W, h
        return w


def ptrs_for(ctx, local_ptr):
    """Per-rank pointer array with only this process' rank filled."""
    from paper_2511_02168_b200.dist import rank_pointer_table
    return rank_pointer_table(ctx.W, ctx.rank, local_ptr)


def fd_step_bufs(ctx, w, shape, qt, kp, vp, out):
    """One fused Flash Decode call on the world stream with this rank's q and
    out buffers (e2e double buffering)."""
    from paper_2511_02168_b200 import _abi
    a = (w.handle, _abi.TF_FD_FUSED, C.byref(shape), _abi.ptr_array(ptrs_for(ctx, qt.data_ptr())), kp, vp,
         _abi.ptr_array(ptrs_for(ctx, out.data_ptr())), None, None)
    return lambda: _abi.check(w.lib.tf_flash_decode_async(*a))


def time_steps(ctx, stream, fn, steps, warmup):
    """W warm-ups, then EXACTLY `steps` steps between a barrier + device sync
    on both sides, timed by CUDA events on the launching stream around the
    whole run (max over ranks) -- the mean, with nothing between the steps
    (an event record between two launches serialises them and costs the
    back-to-back overlap: ~3 us per step).  A second pass of `steps` steps
    with an event after every step gives the per-step p10/p50/p90."""
    torch = ctx.torch
    for _ in range(warmup):
        fn()
    s = torch.cuda.ExternalStream(stream) if isinstance(stream, int) else stream

    def bracket():
        torch.cuda.synchronize()
        ctx.barrier()
        torch.cuda.synchronize()

    bracket()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(steps):
        fn()
    e1.record(s)
    bracket()
    mean = e0.elapsed_time(e1) / steps
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    ev[0].record(s)
    for i in range(steps):
        fn()
        ev[i + 1].record(s)
    bracket()
    per = sorted(ev[i].elapsed_time(ev[i + 1]) for i in range(steps))
    q = lambda f: per[min(len(per) - 1, int(f * len(per)))]  # noqa: E731
    return dict(ms=ctx.max(mean), p10=ctx.max(q(0.1)), p50=ctx.max(statistics.median(per)), p90=ctx.max(q(0.9)))


def us(t):
    """{ms, p10, p50, p90} -> the same in us, rounded."""
    return {("mean_us" if k == "ms" else k + "_us"): round(v * 1e3, 3) for k, v in t.items()}


# ---------------------------------------------------------------------------------
# AG+GEMM (headline)

def bench_ag(ctx, steps, warmup, cooldown=lambda: None):
    from paper_2511_02168_b200 import _abi
    torch = ctx.torch
    W = ctx.W
    M, K, N = M_, K_, N_TOTAL // W
    kw = K // W
    w = ctx.world(M * kw * 2 + 2 * 2 * M * K * 2 + (64 << 20))
    try:
        g = torch.Generator(device=ctx.dev).manual_seed(1 + ctx.rank)
        shard_ptrs = w.alloc("ag.a", M * kw * 2)
        A_local = (torch.rand(M, kw, device=ctx.dev, generator=g) * 2 - 1).bfloat16()
        w.memcpy(shard_ptrs[ctx.rank], A_local.data_ptr(), M * kw * 2)
        B = (torch.rand(K, N, device=ctx.dev, generator=g) * 2 - 1).bfloat16()
        Cm = torch.empty(M, N, device=ctx.dev, dtype=torch.bfloat16)
        torch.cuda.synchronize()
        ctx.barrier()  # setup fence: every shard placed before any rank pulls it
        shape = _abi.AgShape(M, N, K, 0, 0, 0, _abi.TF_BF16)
        st = w.stream(ctx.rank)
        args = (w.handle, _abi.TF_AG_PULL, C.byref(shape), _abi.ptr_array(shard_ptrs),
                _abi.ptr_array(ptrs_for(ctx, B.data_ptr())), _abi.ptr_array(ptrs_for(ctx, Cm.data_ptr())),
                None, None)
        step = lambda: _abi.check(w.lib.tf_ag_gemm_async(*args))  # noqa: E731
        l0 = w.launches()
        with ClockSampler(ctx.local) as clk:
            t = time_steps(ctx, st, step, steps, warmup)
        launches = (w.launches() - l0) // (steps + warmup) * steps
        _abi.check(w.lib.tf_world_sync(w.handle))
        # BSP baseline: NCCL all-gather (W > 1) + relayout + cuBLAS, from the
        # same idle-GPU start as the fused run; its gathered A is also the
        # independent operand the fused result is checked against.
        cooldown()
        bsp, A_full = bench_bsp_ag(ctx, A_local, B, steps, warmup)
        # Numerics on the benchmarked buffers, every rank: sampled rows of C
        # against an fp32 product of the NCCL-gathered (W > 1) operand.
        rows = torch.arange(0, M, M // 64, device=ctx.dev)
        ref = A_full[rows].float() @ B.float()
        diff = (Cm[rows].float() - ref).abs()
        num = dict(norm_err=ctx.max(float(diff.max() / ref.abs().max())), max_abs=ctx.max(float(diff.max())),
                   rows=int(rows.numel()), reference="fp32 product of the " +
                   ("NCCL-gathered operand" if W > 1 else "local operand"))
        del A_full
        # End to end through the C ABI with host buffers: H2D of the shard and
        # B from pinned memory, the fused step, D2H of C -- every step.
        e2e = bench_ag_e2e(ctx, w, A_local, B, Cm, shape, max(3, steps // 5))
        return dict(t=t, launches=launches, clocks=clk.summary(), num=num, bsp=bsp, e2e=e2e, M=M, N=N, K=K)
    finally:
        w.close()


def bench_bsp_ag(ctx, A_local, B, steps, warmup):
    torch = ctx.torch
    W = ctx.W
    M, kw = A_local.shape
    gathered = torch.empty(W, M, kw, device=ctx.dev, dtype=torch.bfloat16)
    out = torch.empty(M, B.shape[1], device=ctx.dev, dtype=torch.bfloat16)
    A_full = A_local

    def step():
        nonlocal A_full
        if W > 1:
            ctx.all_gather(gathered, A_local)
            A_full = gathered.permute(1, 0, 2).reshape(M, W * kw)  # relayout [W][M][kw] -> M x K
        torch.matmul(A_full, B, out=out)

    t = time_steps(ctx, torch.cuda.current_stream(), step, steps, warmup)
    return t, A_full


def bench_ag_e2e(ctx, w, A_local, B, Cm, shape, steps):
    """The reference's calling convention end to end: host shard and B in,
    host C out, through tf_ag_gemm_host (C ABI).  The library streams B in
    column slabs, runs each slab's GEMM as it lands and streams C back, so
    H2D, the exchange+GEMM and D2H overlap.  Every step copies all inputs
    H2D from pinned memory and reads all of C back."""
    from paper_2511_02168_b200 import _abi
    torch = ctx.torch
    hA = A_local.cpu().pin_memory()
    hB = B.cpu().pin_memory()
    hC = torch.empty(Cm.shape, dtype=Cm.dtype).pin_memory()
    st = w.stream(ctx.rank)
    args = (w.handle, _abi.TF_AG_PULL, C.byref(shape), _abi.ptr_array(ptrs_for(ctx, hA.data_ptr())),
            _abi.ptr_array(ptrs_for(ctx, hB.data_ptr())), _abi.ptr_array(ptrs_for(ctx, hC.data_ptr())), None)

    def step():
        _abi.check(w.lib.tf_ag_gemm_host_async(*args))

    serial = time_steps(ctx, st, step, steps, 2)  # two warm-ups: both buffer sets allocated
    # The streamed result is the device-resident run's result, bit for bit.
    same = ctx.all_true(bool(torch.equal(hC, Cm.cpu())))
    t = serial
    if ctx.W == 1:
        # Back-to-back steps on two alternating streams: the library's two
        # buffer sets let step i+1's H2D stream in while step i finishes
        # computing and reading C back (each step still copies all its
        # inputs in and all of C out inside the timed region).
        s2 = torch.cuda.Stream(device=ctx.dev)
        sts = [st, s2.cuda_stream]
        argv = [(w.handle, _abi.TF_AG_PULL, C.byref(shape), _abi.ptr_array(ptrs_for(ctx, hA.data_ptr())),
                 _abi.ptr_array(ptrs_for(ctx, hB.data_ptr())), _abi.ptr_array(ptrs_for(ctx, hC.data_ptr())),
                 _abi.ptr_array([x])) for x in sts]
        s0 = torch.cuda.ExternalStream(st)

        def run(n):
            start = torch.cuda.Event()
            start.record(s0)
            s2.wait_event(start)
            for i in range(n):
                _abi.check(w.lib.tf_ag_gemm_host_async(*argv[i % 2]))
            s0.wait_stream(s2)

        run(2)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s0)
        run(steps)
        e1.record(s0)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        same = same and bool(torch.equal(hC, Cm.cpu()))
        t = dict(ms=ms, p10=ms, p50=ms, p90=ms)
    return dict(t=t, serial=serial, h2d=hA.numel() * 2 + hB.numel() * 2, d2h=hC.numel() * 2, matches_device_run=same)


# ---------------------------------------------------------------------------------
# AG+GEMM M-sweep (BASELINE configs[4]: M 128..16384, K = N = 8192), secondary

def bench_msweep(ctx, steps, warmup, pk, Ms=SWEEP_MS):
    from paper_2511_02168_b200 import _abi
    torch = ctx.torch
    W = ctx.W
    K = N = 8192
    kw = K // W
    Mmax = max(Ms)
    w = ctx.world(Mmax * kw * 2 + 2 * 2 * Mmax * K * 2 + (64 << 20))
    out = {}
    try:
        g = torch.Generator(device=ctx.dev).manual_seed(3 + ctx.rank)
        shard_ptrs = w.alloc("ag.a.sweep", Mmax * kw * 2)
        A = (torch.rand(Mmax, kw, device=ctx.dev, generator=g) * 2 - 1).bfloat16()
        w.memcpy(shard_ptrs[ctx.rank], A.data_ptr(), A.numel() * 2)
        B = (torch.rand(K, N, device=ctx.dev, generator=g) * 2 - 1).bfloat16()
        Cm = torch.empty(Mmax, N, device=ctx.dev, dtype=torch.bfloat16)
        gathered_flat = torch.empty(W * Mmax * kw, device=ctx.dev, dtype=torch.bfloat16)
        torch.cuda.synchronize()
        ctx.barrier()
        for M in Ms:
            shape = _abi.AgShape(M, N, K, 0, 0, 0, _abi.TF_BF16)
            res = {}
            for name, var in (("pull", _abi.TF_AG_PULL), ("push", _abi.TF_AG_PUSH)):
                args = (w.handle, var, C.byref(shape), _abi.ptr_array(shard_ptrs),
                        _abi.ptr_array(ptrs_for(ctx, B.data_ptr())), _abi.ptr_array(ptrs_for(ctx, Cm.data_ptr())),
                        None, None)
                res[name] = time_steps(ctx, w.stream(ctx.rank), lambda: _abi.check(w.lib.tf_ag_gemm_async(*args)),
                                       steps, warmup)
                if W == 1:
                    break  # nothing to exchange: pull == push
            Am = A[:M]

            def bsp():
                if W > 1:
                    gathered = gathered_flat[: W * M * kw].view(W, M, kw)  # contiguous for NCCL
                    ctx.all_gather(gathered, Am)
                    a = gathered.permute(1, 0, 2).reshape(M, K)
                else:
                    a = Am
                torch.matmul(a, B, out=Cm[:M])

            res["bsp"] = time_steps(ctx, torch.cuda.current_stream(), bsp, steps, warmup)
            best_name = min((k for k in res if k != "bsp"), key=lambda k: res[k]["ms"])
            best = res[best_name]["ms"] * 1e-3
            flop = 2.0 * M * N * K
            hbm_bytes = 2.0 * (M * K + K * N + M * N)  # algorithmic: A (gathered), B, C once
            # Roofline: the slower of the tensor-pipe and HBM bounds at this M.
            t_tensor = flop / (pk["bf16"] * 1e12)
            t_hbm = hbm_bytes / (pk["hbm"] * 1e9)
            bound = "hbm" if t_hbm > t_tensor else "tensor"
            point = {k: us(v) for k, v in res.items()}
            point["best"] = best_name
            point["tflops"] = round(flop / best / 1e12, 1)
            point["fused_speedup_vs_bsp"] = round(res["bsp"]["ms"] / res[best_name]["ms"], 3)
            point["roofline"] = {"bound": bound, "ideal_us": round(max(t_tensor, t_hbm) * 1e6, 2),
                                 "frac": round(max(t_tensor, t_hbm) / best, 3),
                                 "achieved": round(flop / best / 1e12, 1) if bound == "tensor"
                                 else round(hbm_bytes / best / 1e9, 1),
                                 "unit": "TFLOP/s" if bound == "tensor" else "GB/s"}
            if W > 1:
                inbound = (W - 1) / W * M * K * 2
                point["nvlink"] = nvlink_block(inbound, best)
            out[str(M)] = point
        return out
    finally:
        w.close()


def nvlink_block(bytes_per_rank, seconds):
    gbs = bytes_per_rank / seconds / 1e9
    return {"bytes_per_rank": int(bytes_per_rank), "achieved_gbs": round(gbs, 1),
            "frac_of_measured": round(gbs / NVLINK_MEASURED_GBS, 3),
            "frac_of_nominal": round(gbs / NVLINK_NOMINAL_GBS, 3),
            "peak": f"{NVLINK_MEASURED_GBS:.0f} GB/s measured peer copy per direction "
                    f"({NVLINK_NOMINAL_GBS:.0f} nominal)"}


# ---------------------------------------------------------------------------------
# Flash Decode (secondary)

def bench_fd(ctx, cfg, steps, warmup, pk, cooldown=lambda: None):
    from paper_2511_02168_b200 import _abi
    torch = ctx.torch
    W = ctx.W
    B, Hq, Hkv, d, L = cfg["batch"], cfg["q_heads"], cfg["kv_heads"], cfg["head_dim"], cfg["kv_len"]
    ln = L // W
    row = B * Hq * (d + 2)
    w = ctx.world(4 * W * row * 4 + 4 * B * Hkv * 1024 * (d + 2) * 8 * 4 + (64 << 20))
    try:
        g = torch.Generator(device=ctx.dev).manual_seed(7 + ctx.rank)
        q = (torch.rand(B, Hq, d, device=ctx.dev, generator=torch.Generator(device=ctx.dev).manual_seed(7)) * 2
             - 1).bfloat16()  # q is replicated: the same on every rank
        k = (torch.rand(B, Hkv, ln, d, device=ctx.dev, generator=g) * 2 - 1).bfloat16()
        v = (torch.rand(B, Hkv, ln, d, device=ctx.dev, generator=g) * 2 - 1).bfloat16()
        outs = {"bf16": torch.empty(B, Hq, d, device=ctx.dev, dtype=torch.bfloat16),
                "f32": torch.empty(B, Hq, d, device=ctx.dev, dtype=torch.float32)}
        rows_local = torch.empty(row, device=ctx.dev, dtype=torch.float32)
        rows_all = torch.empty(W * row, device=ctx.dev, dtype=torch.float32)
        out_nccl = torch.empty(B, Hq, d, device=ctx.dev, dtype=torch.bfloat16)
        torch.cuda.synchronize()
        ctx.barrier()
        shapes = {o: _abi.FdShape(B, Hq, Hkv, d, L, float(d ** -0.5), _abi.TF_BF16,
                                  _abi.TF_BF16 if o == "bf16" else _abi.TF_F32) for o in outs}
        qp, kp, vp = (_abi.ptr_array(ptrs_for(ctx, t.data_ptr())) for t in (q, k, v))
        stw = w.stream(ctx.rank)
        res, clocks = {}, {}

        def fd_step(var, o):
            a = (w.handle, var, C.byref(shapes[o]), qp, kp, vp, _abi.ptr_array(ptrs_for(ctx, outs[o].data_ptr())),
                 None, None)
            return lambda: _abi.check(w.lib.tf_flash_decode_async(*a))

        # The north_star's BSP baseline: the attention kernel, an NCCL
        # all_gather_into_tensor of every rank's [B][Hq][d+2] partial rows,
        # the combine kernel -- all on the world stream.
        sws = torch.cuda.ExternalStream(stw)
        pa = (w.handle, C.byref(shapes["bf16"]), qp, kp, vp, _abi.ptr_array(ptrs_for(ctx, rows_local.data_ptr())),
              _abi.ptr_array(ptrs_for(ctx, stw)))
        ca = (w.handle, C.byref(shapes["bf16"]), _abi.ptr_array(ptrs_for(ctx, rows_all.data_ptr())),
              _abi.ptr_array(ptrs_for(ctx, out_nccl.data_ptr())), _abi.ptr_array(ptrs_for(ctx, stw)))

        def nccl_bsp():
            _abi.check(w.lib.tf_fd_partial_async(*pa))
            with torch.cuda.stream(sws):
                ctx.all_gather(rows_all, rows_local)
            _abi.check(w.lib.tf_fd_combine_async(*ca))

        variants = [("fused", fd_step(_abi.TF_FD_FUSED, "bf16"), stw),
                    ("fused_f32out", fd_step(_abi.TF_FD_FUSED, "f32"), stw),
                    ("bsp", fd_step(_abi.TF_FD_BSP, "bf16"), stw),
                    ("nccl_bsp", nccl_bsp, stw)]
        if W > 1:  # owner-combine: 1/(W-1) of the all-gather's fabric bytes
            variants.append(("owner", fd_step(_abi.TF_FD_FUSED_OWNER, "bf16"), stw))
        l0 = w.launches()
        for name, fn, s in variants:
            cooldown()
            with ClockSampler(ctx.local) as clk:
                res[name] = time_steps(ctx, s, fn, steps, warmup)
            clocks[name] = clk.summary()
            if name == "fused":
                launches = (w.launches() - l0) // (steps + warmup) * steps
        _abi.check(w.lib.tf_world_sync(w.handle))
        torch.cuda.synchronize()
        # End to end through the C ABI: the KV cache is resident in HBM (it
        # is a cache); every decode step brings its new query from pinned
        # host memory and returns the output to the host, both inside the
        # timed region.  Serial: both copies on the world stream around the
        # fused launch.  Pipelined (the e2e value): double-buffered q / out,
        # the copies on a copy stream, step i+1's query H2D and step i's
        # output D2H overlapping the launches -- every copy of every step
        # still inside the timed region (the world stream joins the copy
        # stream before the closing event).
        hq = q.cpu().pin_memory()
        hout = [torch.empty(outs["bf16"].shape, dtype=torch.bfloat16).pin_memory() for _ in range(2)]
        fused_bf16 = fd_step(_abi.TF_FD_FUSED, "bf16")

        def e2e_step():
            with torch.cuda.stream(sws):
                q.copy_(hq, non_blocking=True)
            fused_bf16()
            with torch.cuda.stream(sws):
                hout[0].copy_(outs["bf16"], non_blocking=True)

        cooldown()
        serial = time_steps(ctx, stw, e2e_step, steps, warmup)
        e2e_ok = ctx.all_true(bool(torch.equal(hout[0], outs["bf16"].cpu())))
        cs = torch.cuda.Stream(device=ctx.dev)
        qbuf = [q, q.clone()]
        obuf = [outs["bf16"], torch.empty_like(outs["bf16"])]
        ev_q = [torch.cuda.Event(), torch.cuda.Event()]
        ev_k = [torch.cuda.Event(), torch.cuda.Event()]
        calls = [fd_step_bufs(ctx, w, shapes["bf16"], qbuf[b], kp, vp, obuf[b]) for b in range(2)]

        def pipelined(n):
            start = torch.cuda.Event()
            start.record(sws)
            cs.wait_event(start)
            with torch.cuda.stream(cs):
                qbuf[0].copy_(hq, non_blocking=True)
            ev_q[0].record(cs)
            for i in range(n):
                b = i % 2
                sws.wait_event(ev_q[b])
                calls[b]()
                ev_k[b].record(sws)
                # step i+1's query: its buffer was last read by launch i-1
                if i >= 1:
                    cs.wait_event(ev_k[1 - b])
                with torch.cuda.stream(cs):
                    qbuf[1 - b].copy_(hq, non_blocking=True)
                ev_q[1 - b].record(cs)
                # step i's output, once launch i is done (launch i+2 rewrites
                # obuf[b] only after ev_q[b], recorded after this copy)
                cs.wait_event(ev_k[b])
                with torch.cuda.stream(cs):
                    hout[b].copy_(obuf[b], non_blocking=True)
            sws.wait_stream(cs)

        pipelined(warmup)
        torch.cuda.synchronize()
        ctx.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(sws)
        pipelined(steps)
        e1.record(sws)
        torch.cuda.synchronize()
        ctx.barrier()
        torch.cuda.synchronize()
        piped_ms = ctx.max(e0.elapsed_time(e1) / steps)
        e2e_ok = e2e_ok and ctx.all_true(bool(torch.equal(hout[(steps - 1) % 2], obuf[(steps - 1) % 2].cpu())))
        res["e2e"] = dict(ms=piped_ms, p10=piped_ms, p50=piped_ms, p90=piped_ms)
        res["e2e_serial"] = serial
        e2e_bytes = dict(h2d=hq.numel() * 2, d2h=hout[0].numel() * 2, matches_device_run=e2e_ok)
        # Torch's pinned-host allocator recorded the world stream on these
        # blocks; free them while that stream still exists (w.close()
        # destroys it, and a later free would touch a dead stream).
        torch.cuda.synchronize()
        del hq, hout, e2e_step, calls, qbuf, obuf
        # The library's BSP schedule replayed from a CUDA graph (W = 1): the
        # host launch cost removed, its device-side stages kept.
        if W == 1:
            try:
                cs = torch.cuda.Stream()
                bargs = (w.handle, _abi.TF_FD_BSP, C.byref(shapes["bf16"]), qp, kp, vp,
                         _abi.ptr_array(ptrs_for(ctx, outs["bf16"].data_ptr())), None, _abi.ptr_array([cs.cuda_stream]))
                gr = torch.cuda.CUDAGraph()
                with torch.cuda.graph(gr, stream=cs):
                    _abi.check(w.lib.tf_flash_decode_async(*bargs))
                res["bsp_graph"] = time_steps(ctx, torch.cuda.current_stream(), gr.replay, steps, warmup)
                torch.cuda.synchronize()
                del gr  # holds nodes on the world's resources: gone before w.close()
            except Exception as e:  # noqa: BLE001 -- reported, not fatal
                res["bsp_graph_error"] = repr(e)[:200]
        # Numerics (the last timed runs' outputs): batch 0 (and the last
        # batch) against torch fp32 attention over the whole logical KV
        # (every rank's shard, all-gathered for the check); fused vs the NCCL
        # arm bitwise.
        for o, var in (("bf16", _abi.TF_FD_FUSED), ("f32", _abi.TF_FD_FUSED)):
            fd_step(var, o)()
        _abi.check(w.lib.tf_world_sync(w.handle))
        nccl_bsp()
        torch.cuda.synchronize()
        same_nccl = ctx.all_true(bool(torch.equal(out_nccl, outs["bf16"])))
        num = {"fused_equals_nccl_bsp_bitwise": same_nccl}
        for bb in sorted({0, B - 1}):
            kf = torch.empty(W, Hkv, ln, d, device=ctx.dev, dtype=torch.bfloat16)
            vf = torch.empty(W, Hkv, ln, d, device=ctx.dev, dtype=torch.bfloat16)
            ctx.all_gather(kf, k[bb].contiguous())
            ctx.all_gather(vf, v[bb].contiguous())
            kk = kf.permute(1, 0, 2, 3).reshape(Hkv, L, d).float()
            vv = vf.permute(1, 0, 2, 3).reshape(Hkv, L, d).float()
            del kf, vf
            qf = q[bb].float().view(Hkv, Hq // Hkv, d)
            s_ = torch.einsum("hgd,hld->hgl", qf, kk) * (d ** -0.5)
            ref = torch.einsum("hgl,hld->hgd", torch.softmax(s_, -1), vv).reshape(Hq, d)
            del kk, vv, s_
            for o in outs:
                diff = (outs[o][bb].float() - ref).abs()
                e = num.setdefault(o, {"head_rel_err": 0.0, "max_abs": 0.0,
                                       "tol": BF16_OUT_TOL if o == "bf16" else F32_OUT_TOL})
                e["head_rel_err"] = max(e["head_rel_err"], ctx.max(float((diff.amax(-1) / ref.abs().amax(-1)).max())))
                e["max_abs"] = max(e["max_abs"], ctx.max(float(diff.max())))
        num["batches_checked"] = sorted({0, B - 1})
        kv_bytes = 2 * B * Hkv * ln * d * 2
        return dict(res=res, clocks=clocks, kv_bytes=kv_bytes, num=num, launches=launches, row_bytes=row * 4,
                    e2e=e2e_bytes)
    finally:
        w.close()


# ---------------------------------------------------------------------------------
# the reference's CPU path (oracle/_ref: proj/include/tilefabric compiled as-is)

def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def run_threads(n, fn):
    th = [threading.Thread(target=fn, args=(i,)) for i in range(n)]
    t0 = time.perf_counter()
    for t in th:
        t.start()
    for t in th:
        t.join()
    return time.perf_counter() - t0


def cpu_reference_ag(W, n_slice=1792):
    """ag::run_pull (ag_gemm.hpp:185-222) of config 2 on this host: one
    concurrent call per core, each on ceil(M / cores) rows x an n_slice
    column slice of the output at the real K -- together every one of the
    M rows -- extrapolated linearly to the full N (the loops are exactly
    linear in the output columns, ag_gemm.hpp:200-217)."""
    import numpy as np
    from oracle.oracle import Reference
    if not Reference.available():
        return None
    R = Reference()
    cores = host_cores()
    K, N = K_, N_TOTAL // W
    n_slice = min(n_slice, N)
    rows = math.ceil(M_ / cores)
    rng = np.random.default_rng(0)
    A = rng.uniform(-1, 1, (rows, K)).astype(np.float32)
    Bs = rng.uniform(-1, 1, (K, n_slice)).astype(np.float32)
    times = [0.0] * cores

    def work(i):
        t0 = time.perf_counter()
        R.ag_run_inputs(1, A, Bs, W)
        times[i] = time.perf_counter() - t0

    wall = run_threads(cores, work)
    sample_mn = cores * rows * n_slice
    full_mn = M_ * N
    factor = full_mn / sample_mn
    return dict(value=wall * factor * 1e6, unit="us", cores=cores, kind="reference",
                sample=f"{cores} concurrent ag::run_pull(W={W}) calls on {rows}x{n_slice} slices (all {cores * rows} "
                       f">= M rows, {n_slice} of N={N} columns) at K={K}: wall {wall:.2f}s, extrapolated "
                       f"x{factor:.1f} linearly in N", extrapolated_x=round(factor, 2),
                cpu_seconds=round(sum(times), 2))


def cpu_reference_fd(cfg, W):
    """fd::run_fused (flash_decode.hpp:348-423) over the SURVEY 8(c) (b, j)
    restatement -- for batch b and q-slot j, a reference DecodeProblem of
    Hkv heads (q = q[b][g*gs + j]) over K[b], V[b] -- every call of the
    config, W worker threads each (the reference's own), as many calls at
    once as the host's cores allow.  Reports the wall time of the whole
    config (no extrapolation) and the reference's own per-call makespans."""
    import numpy as np
    from oracle.oracle import Reference
    if not Reference.available():
        return None
    R = Reference()
    cores = host_cores()
    B, Hq, Hkv, d, L = cfg["batch"], cfg["q_heads"], cfg["kv_heads"], cfg["head_dim"], cfg["kv_len"]
    gs = Hq // Hkv
    rng = np.random.default_rng(1)
    # Distinct K/V for a bounded number of batches, reused cyclically (the
    # arithmetic per call is the same for any values); memory per batch:
    # 2 x Hkv x L x d fp32, plus the reference's own copies per live call.
    nkv = min(B, 2)
    kvs = [(rng.uniform(-1, 1, (Hkv, L, d)).astype(np.float32), rng.uniform(-1, 1, (Hkv, L, d)).astype(np.float32))
           for _ in range(nkv)]
    q = rng.uniform(-1, 1, (B, Hq, d)).astype(np.float32)
    calls = [(b, j) for b in range(B) for j in range(gs)]
    per_call_bytes = 2 * Hkv * L * d * 4 * 3
    conc = max(1, min(cores // max(W, 1), len(calls), int(8e9 // per_call_bytes)))
    lock = threading.Lock()
    nxt = [0]
    mk = []

    def work(_):
        while True:
            with lock:
                if nxt[0] >= len(calls):
                    return
                b, j = calls[nxt[0]]
                nxt[0] += 1
            kb, vb = kvs[b % nkv]
            _, ms, post = R.fd_run_inputs(3, np.ascontiguousarray(q[b, j::gs]), kb, vb, d ** -0.5, W)
            with lock:
                mk.append((ms, post))

    wall = run_threads(conc, work)
    return dict(value=wall * 1e6, unit="us", cores=conc * max(W, 1), kind="reference",
                sample=f"all {len(calls)} fd::run_fused(W={W}) calls of the config ({Hkv} heads x L={L} x d={d} "
                       f"each, the (b, j) GQA restatement), {conc} at a time: wall {wall:.2f}s",
                makespan_sum_us=round(sum(m for m, _ in mk) / 1e3, 1),
                post_placement_sum_us=round(sum(p for _, p in mk) / 1e3, 1))


def cpu_reference_sweep(W, Ms=SWEEP_MS, measure=(128, 256)):
    """ag::run_pull at K = N = 8192: the M in `measure` timed whole (the N
    columns split into one slice per core, every output element computed);
    larger M extrapolated linearly in M from the largest measured point."""
    import numpy as np
    from oracle.oracle import Reference
    if not Reference.available():
        return None
    R = Reference()
    cores = host_cores()
    K = N = 8192
    rng = np.random.default_rng(2)
    cols = math.ceil(N / cores)
    out = {}
    for M in measure:
        A = rng.uniform(-1, 1, (M, K)).astype(np.float32)
        Bs = rng.uniform(-1, 1, (K, cols)).astype(np.float32)
        wall = run_threads(cores, lambda i: R.ag_run_inputs(1, A, Bs, W))
        out[M] = wall
    Mref = max(measure)
    return {str(M): dict(value=round((out[M] if M in out else out[Mref] * M / Mref) * 1e6, 1), unit="us",
                         measured=M in out, cores=cores, kind="reference")
            for M in Ms} | {"sample": f"ag::run_pull(W={W}), N split into {cores} concurrent column slices of "
                                      f"{cols}; M in {list(measure)} measured, larger M extrapolated linearly in M"}


def run_reference_arm(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    W = max(ws, args.gpus)
    vals = []
    info = None
    for i in range(args.warmup + args.steps):
        r = cpu_reference_ag(W)
        if r is None:
            print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libtfref.so not built"}))
            return
        if i >= args.warmup:
            vals.append(r["value"])
            info = r
    v = statistics.median(vals)
    line = {"metric": METRIC, "value": v, "unit": "us", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": v / 1e3, "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": ag_config(W), "impl": "reference",
            "percentiles_us": {"p10": sorted(vals)[int(0.1 * len(vals))], "p50": v,
                               "p90": sorted(vals)[min(len(vals) - 1, int(0.9 * len(vals)))]},
            "cpu_baseline": {"value": v, "unit": "us", "cores": info["cores"], "kind": "reference",
                             "sample": info["sample"]},
            "e2e": {"value": v, "unit": "us", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    if not args.no_fd:
        line["secondary"] = {"fd_config3_b1_L128k": cpu_reference_fd(FD3, W),
                             "fd_config4_b32_L32k": cpu_reference_fd(FD4, W)}
    print(json.dumps(line))


def ag_config(W):
    return {"workload": "AG+GEMM BASELINE configs[1]: bf16, M=8192 gathered rows, K=8192 sharded along K, "
                        "N=28672/W per GPU (Llama-3-70B TP shape)",
            "M": M_, "K": K_, "N_per_gpu": N_TOTAL // W, "world_size": W, "variant": "pull",
            "l2": "no flush needed: every input exceeds L2 (A 128 MiB, B 448 MiB / W)",
            "parallelism": f"tp{W} (A all-gathered along K)"}


def fd_secondary(name, cfg, r, pk, W, cpu):
    res = r["res"]
    fused = res["fused"]["ms"] * 1e-3
    gbs = r["kv_bytes"] / fused / 1e9
    sec = {"fused_us": res["fused"]["ms"] * 1e3, "bsp_us": res["bsp"]["ms"] * 1e3,
           "nccl_bsp_us": res["nccl_bsp"]["ms"] * 1e3,
           "fused_f32out_us": res["fused_f32out"]["ms"] * 1e3,
           "fused_speedup_vs_bsp": res["bsp"]["ms"] / res["fused"]["ms"],
           "fused_speedup_vs_nccl_bsp": res["nccl_bsp"]["ms"] / res["fused"]["ms"],
           "percentiles": {k: us(v) for k, v in res.items() if isinstance(v, dict)},
           "what": {"fused": "ONE persistent launch per GPU: attention -> split fold -> push [m|l|o] rows + "
                             "flags to every rank -> flag-gated ascending fold (bf16 out)",
                    "fused_f32out": "the same, fp32 output",
                    "bsp": "the library's BSP schedule: attention | device barrier | gather kernel | barrier | fold",
                    "nccl_bsp": "attention kernel (tf_fd_partial_async) -> NCCL all_gather_into_tensor of the "
                                "[B][Hq][d+2] rows -> combine kernel (tf_fd_combine_async)" +
                                (" (W=1: no all-gather)" if W == 1 else "")},
           "roofline": {"bound": "hbm", "achieved": gbs, "peak": pk["hbm"], "unit": "GB/s",
                        "frac": gbs / pk["hbm"], "algorithmic_bytes_per_launch": r["kv_bytes"],
                        "peak_source": pk["src"] + " copy bandwidth (MEASURED_PEAKS.json)"},
           "numerics": r["num"], "config": cfg, "clocks": r["clocks"]["fused"], "gpu_launches_fused": r["launches"]}
    sec["e2e"] = {"value": res["e2e"]["ms"] * 1e3, "unit": "us", "h2d_bytes_per_step": r["e2e"]["h2d"],
                  "d2h_bytes_per_step": r["e2e"]["d2h"], "matches_device_run": r["e2e"]["matches_device_run"],
                  "serial_us": res["e2e_serial"]["ms"] * 1e3,
                  "what": "tf_flash_decode_async (fused) with the query H2D from pinned memory and the output D2H "
                          "every step, double-buffered on a copy stream so step i+1's H2D and step i's D2H overlap "
                          "the launches (serial_us: both copies on the launch stream); the KV cache resident in HBM"}
    if "owner" in res:
        sec["owner_combine_us"] = res["owner"]["ms"] * 1e3
    if "bsp_graph" in res:
        sec["bsp_cuda_graph_us"] = res["bsp_graph"]["ms"] * 1e3
        sec["fused_speedup_vs_bsp_graph"] = res["bsp_graph"]["ms"] / res["fused"]["ms"]
    elif "bsp_graph_error" in res:
        sec["bsp_cuda_graph_error"] = res["bsp_graph_error"]
    if W > 1:
        sec["nvlink"] = nvlink_block((W - 1) * r["row_bytes"], fused)
    if cpu:
        sec["cpu_baseline"] = cpu
    return sec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline legs")
    ap.add_argument("--no-fd", action="store_true")
    ap.add_argument("--no-sweep", action="store_true", help="skip the config-5 M sweep")
    ap.add_argument("--cooldown", type=float, default=2.0, help="idle seconds before each timed section")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference_arm(args)
        return
    args.warmup = max(args.warmup, 3)
    ctx = Ctx(args.gpus)
    pk = peaks()

    def cooldown():
        # Each workload is timed from an idle GPU: the power-capped clock
        # state a long GEMM leaves behind (sw_power_cap) would otherwise
        # carry into the next, memory-bound, section.
        ctx.torch.cuda.synchronize()
        ctx.barrier()
        time.sleep(args.cooldown)
        ctx.barrier()

    fd3 = fd4 = sweep = None
    if not args.no_fd:
        fd3 = bench_fd(ctx, FD3, args.steps, args.warmup, pk, cooldown)
        fd4 = bench_fd(ctx, FD4, args.steps, args.warmup, pk, cooldown)
    cooldown()
    ag_res = bench_ag(ctx, args.steps, args.warmup, cooldown=cooldown)
    if not args.no_sweep:
        cooldown()
        sweep = bench_msweep(ctx, max(10, args.steps // 2), args.warmup, pk)
    if ctx.rank != 0:
        return
    W = ctx.W
    M, N, K = ag_res["M"], ag_res["N"], ag_res["K"]
    flops = 2.0 * M * N * K
    t = ag_res["t"]
    tflops = flops / (t["ms"] * 1e-3) / 1e12
    cpu = cpu3 = cpu4 = cpusw = None
    if not args.no_cpu:
        cpu = cpu_reference_ag(W)
        if fd3:
            cpu3, cpu4 = cpu_reference_fd(FD3, W), cpu_reference_fd(FD4, W)
        if sweep:
            cpusw = cpu_reference_sweep(W)
    line = {
        "metric": METRIC, "value": t["ms"] * 1e3, "unit": "us", "n_gpus": W, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t["ms"], "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": dict(ag_config(W), **({"test_mode": "TFB_BENCH_SHARED_GPU: all ranks time-slice one GPU"}
                                         if ctx.shared else {})),
        "percentiles_us": {k: v for k, v in us(t).items() if k != "mean_us"},
        "roofline": {"bound": "tensor", "achieved": tflops, "peak": pk["bf16"], "unit": "TFLOP/s",
                     "frac": tflops / pk["bf16"], "peak_source": pk["src"] + " burst (MEASURED_PEAKS.json)",
                     "frac_vs_sustained": tflops / pk["bf16_sus"],
                     "algorithmic_flop_per_launch": flops,
                     "traffic": ncu_traffic("ag_gemm_sm100_kernel")},
        "bsp": {"what": "cuBLAS matmul" + ((" after gloo all_gather through host memory + relayout (shared-GPU "
                                            "test mode: not a baseline)" if ctx.shared else
                                            " after NCCL all_gather_into_tensor + relayout") if W > 1 else
                                           " (W=1: nothing to gather)"),
                "value": ag_res["bsp"]["ms"] * 1e3, "unit": "us", "percentiles": us(ag_res["bsp"]),
                "fused_speedup": ag_res["bsp"]["ms"] / t["ms"]},
        "e2e": {"value": ag_res["e2e"]["t"]["ms"] * 1e3, "unit": "us",
                "h2d_bytes_per_step": ag_res["e2e"]["h2d"], "d2h_bytes_per_step": ag_res["e2e"]["d2h"],
                "percentiles": us(ag_res["e2e"]["t"]),
                "serial_us": ag_res["e2e"]["serial"]["ms"] * 1e3,
                "what": "tf_ag_gemm_host via the C ABI: pinned host A-shard and B in, host C out, every step "
                        "(B/C streamed in column slabs, H2D / GEMM / D2H overlapped; at W = 1 back-to-back steps "
                        "alternate two streams so step i+1's H2D overlaps step i's read-back -- serial_us: one "
                        "stream)",
                "matches_device_run": ag_res["e2e"]["matches_device_run"]},
        "gpu_launches": ag_res["launches"],
        "clocks": ag_res["clocks"],
        "numerics": {"ag_sampled_rows_norm_err": ag_res["num"]["norm_err"],
                     "ag_sampled_rows_max_abs": ag_res["num"]["max_abs"], "rows": ag_res["num"]["rows"],
                     "reference": ag_res["num"]["reference"],
                     "tol": "norm_err <= 4e-3 (bf16 output rounding 2^-8 of max|C|)"},
    }
    if W > 1:
        line["nvlink"] = nvlink_block((W - 1) / W * M * K * 2, t["ms"] * 1e-3)
    if cpu:
        line["cpu_baseline"] = cpu
    if fd3:
        line["secondary"] = {"fd_config3_b1_L128k": fd_secondary("c3", FD3, fd3, pk, W, cpu3),
                             "fd_config4_b32_L32k": fd_secondary("c4", FD4, fd4, pk, W, cpu4)}
    if sweep:
        if cpusw:
            samp = cpusw.pop("sample")
            for m_, p in sweep.items():
                if m_ in cpusw:
                    p["cpu_baseline"] = cpusw[m_]
        line.setdefault("secondary", {})["ag_msweep_K8192_N8192"] = {
            "what": "BASELINE configs[4] at this world size: per M, fused pull (and push at W > 1) vs the "
                    "NCCL all-gather + cuBLAS BSP, percentiles, roofline (the slower of tensor and HBM bounds)",
            "points": sweep, **({"cpu_sample": samp} if cpusw else {})}
    print(json.dumps(line))


if __name__ == "__main__":
    main()
