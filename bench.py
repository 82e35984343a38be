"""Benchmark: semiring matmul & Floyd-Warshall cell-updates/s (n^3/s) vs roofline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload NAME] [--n N]
    python bench.py --impl reference ...      # the reference algorithm on the host CPU

Default workload (BASELINE.json configs[4], the largest single-GPU config):
Floyd-Warshall closure of the n = 32768 anti-distance u16 graph (density 0.02,
w ~ U[1, 1000]); one step = one transitive_closure() of the whole matrix
(copy + closure, exactly the reference's AntidistMatrix.transitive_closure).
For N > 1 the driver launches one rank per GPU under torch.distributed.run;
the closure is row-panel sharded with an NCCL broadcast of each pivot row
panel (paper_1705_08743_b200/sharded.py) -- strong scaling, fixed n.

Reported beside the device-resident throughput (`value`):
  e2e          the same metric through the reference's own call on a host
               numpy array, AntidistMatrix(n, n, 16, arr).transitive_closure()
               .data, per step: one smx_fw_host_u16 call stages the rows in
               through page-locked slots and closes them as they arrive, and
               copies finished rows out while the rest runs (e2e_pinned: the
               same call from page-locked buffers)
  roofline     the dominant kernel (FW phase-3 semiring GEMM, 93+% of the
               step) timed live with CUDA events, against the packed-integer
               issue peak measured in this run by smx_int_issue_probe
  cpu_baseline the reference algorithm (C restatement, all host threads) on a
               bounded sample of the same workload, rank 0 at N = 1 only
  clocks       SM clocks and throttle reasons sampled during the timed region
Inputs (2 GiB at n = 32768) are larger than the 126 MB L2, so no flush is
needed between steps.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

METRIC = "Semiring matmul & Floyd-Warshall cell-updates/s (N^3/s) vs roofline, 1-8 GPU"
UNIT = "cell-updates/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--workload", default="c5_fw_u16")
    ap.add_argument("--n", "--size", dest="n", type=int, default=None,
                    help="override the config's n (testing; --size under torchrun)")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--check", action="store_true",
                    help="N > 1: compare the gathered sharded closure with the single-GPU one")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# --------------------------------------------------------------------------- clocks

class ClockSampler:
    """Samples SM clock and throttle reasons (NVML) while the timed region runs."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.samples, self.reasons, self.ok = [], 0, False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        reasons = [name for bit, name in self.REASONS.items() if self.reasons & bit and bit != 0x1]
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.samples)}


# --------------------------------------------------------------------------- helpers

def cuda_time(fn, iters: int, warmup: int = 1):
    import torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / 1e3 / iters


def graph_time(fn, per: int = 20, iters: int = 20):
    """Device time per call of `fn` with the host out of the loop: `per`
    back-to-back calls captured into one CUDA graph, replayed `iters` times
    between CUDA events on the capturing stream."""
    import torch
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        fn()
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=st):
            for _ in range(per):
                fn()
        g.replay()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(st)
        for _ in range(iters):
            g.replay()
        e.record(st)
        torch.cuda.synchronize()
    return s.elapsed_time(e) / 1e3 / (iters * per)


def measure_issue_peak():
    """Packed-integer issue rate of the semiring inner-loop SASS on every SM."""
    import ctypes
    import torch
    from paper_1705_08743_b200 import _native
    lib = _native.lib()
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    blocks, threads, iters = sms * 8, 256, 4000
    sink = torch.zeros(blocks * threads, dtype=torch.int32, device="cuda")
    out = {}
    for one in (0, 1, 2):
        ipt = ctypes.c_longlong(0)
        fn = lambda: _native.check(lib.smx_int_issue_probe(  # noqa: E731
            sink.data_ptr(), blocks, threads, iters, one, ctypes.byref(ipt),
            _native.stream_ptr()), "probe")
        t = cuda_time(fn, 3, 1)
        out[("pair", "one", "lop3")[one]] = blocks * threads * ipt.value / t
    return out, sms


def load_traffic(workload: str):
    """DRAM bytes per launch of the dominant kernel from the committed ncu
    --set full capture (dram__bytes_read.sum + dram__bytes_write.sum)."""
    p = REPO / "profiles" / "traffic.json"
    if p.exists():
        entry = json.loads(p.read_text()).get(workload)
        if entry:
            return entry["bytes_per_launch"]
    return None


def read_fw_trace(lib, cap):
    """(seconds, cell-updates) of each launch smx_fw_trace_arm recorded."""
    import ctypes
    ms_arr = (ctypes.c_float * cap)()
    cells_arr = (ctypes.c_longlong * cap)()
    cnt = lib.smx_fw_trace_read(ms_arr, cells_arr, cap)
    if cnt < 0:
        raise RuntimeError(f"phase-3 trace read failed ({cnt})")
    return [(ms_arr[i] / 1e3, cells_arr[i]) for i in range(cnt)]


def sharded_roofline(trace, step_secs, n, block, world, dev):
    """Per-rank roofline of the sharded closure: every rank's bulk updates
    (3b) of the first timed step, CUDA-event timed on its main stream inside
    smx_fw_sharded, against that rank's own measured issue ceiling; gathered
    to every rank."""
    import torch
    import torch.distributed as dist
    trace = trace or []
    dom = sum(t for t, _ in trace)
    cells = sum(c for _, c in trace)
    peaks, sms = measure_issue_peak()
    issue = max(peaks["one"], peaks["pair"])
    mine = torch.tensor([cells / dom if dom else 0.0, 2.0 * issue, dom, float(len(trace)), float(cells)],
                        dtype=torch.float64, device=dev)
    every = [torch.zeros_like(mine) for _ in range(world)]
    dist.all_gather(every, mine)
    rows = [r.tolist() for r in every]
    fr = [r[0] / r[1] for r in rows]
    r0 = rows[0]
    return {
        "bound": "int_issue", "achieved": r0[0] / 1e12, "peak": r0[1] / 1e12, "unit": "Tcell/s",
        "frac": fr[0], "traffic": None,
        "kernel": "packed_gemm_u16_kernel (sharded bulk row update 3b, per round)",
        "sms": sms, "issue_rate": r0[1] / 2.0,
        "launches_timed": int(r0[3]), "avg_launch_ms": r0[2] / max(r0[3], 1) * 1e3,
        "share_of_step": r0[2] / step_secs,
        "per_rank_frac": fr, "per_rank_share_of_step": [r[2] / step_secs for r in rows],
        "min_frac": min(fr), "max_frac": max(fr),
        "aggregate_achieved": sum(r[0] for r in rows) / 1e12,
        "peak_source": "measured on every rank: smx_int_issue_probe x 2 cells per u16x2 instruction",
        "algorithmic_bytes_per_launch": (2 * (n // world) * block + 2 * (n // world) * n) * 2,
    }


def full_size_digest(config: str, n: int):
    """The CPU oracle's committed digest of this config's closure at size n
    (tests/golden/config_digests.json; at n = 32768 from
    tools/oracle_full_digest.py), or None."""
    p = REPO / "tests" / "golden" / "config_digests.json"
    if not p.exists():
        return None
    for d in json.loads(p.read_text()):
        if d["config"] == config and d["n"] == n:
            return d
    return None


def sharded_parity(work, cfg, n, world, rank, block, dev, digest):
    """The gathered sharded closure, bit for bit: against the oracle's
    committed sha256 when one exists for (config, n), else against the
    single-GPU closure of the same input (itself oracle-checked)."""
    import hashlib
    import torch
    from paper_1705_08743_b200 import _native, sharded, workloads
    torch.cuda.synchronize()
    full = sharded.gather_rows(work, n, world, block)
    if rank != 0:
        return None
    if digest is not None:
        got = hashlib.sha256(full.cpu().numpy().tobytes()).hexdigest()
        return {"n": n, "bit_exact_vs_oracle_digest": got == digest["output_sha256"],
                "oracle_sha256": digest["output_sha256"][:16]}
    lib = _native.lib()
    (ref_host,) = workloads.make_inputs(cfg, n)
    ref = torch.from_numpy(ref_host).to(dev)
    rws = _native.workspace(lib.smx_fw_workspace_bytes(n, ref.shape[1], cfg.width // 8), dev)
    _native.check(getattr(lib, f"smx_fw_u{cfg.width}")(
        ref.data_ptr(), n, ref.shape[1], _native.SMX_ANTI, rws.data_ptr(), rws.numel(),
        _native.stream_ptr(dev)), "fw")
    return {"n": n, "bit_exact_vs_single_gpu": bool(torch.equal(full, ref))}


# --------------------------------------------------------------------------- CPU (reference algorithm)

# Size of the bounded CPU sample (cpu_baseline and the --impl reference arm):
# about 10 s of the reference algorithm on the box's host cores.  For the
# closure that is the C4 size, n = 8192 (9 s with 16 threads; the 128 MiB
# matrix no longer sits in the host caches, as the full-size one would not:
# 6.1e10 cell-updates/s there against 1.3-2.2e11 at n = 2048 / 4096).
CPU_SAMPLE_N = {"closure": 8192, "mul": 4096, "bool_mul": 1024, "bool_closure": 4096}
REF_MAX_STEPS, REF_MAX_WARMUP = 4, 1


def cpu_fw_sample(n_sample: int, threads: int = 0):
    """The reference algorithm (C restatement of _close_vector, all host
    threads) on the c5 generator at n_sample: returns (cells/s, seconds, out)."""
    import oracle
    from paper_1705_08743_b200 import workloads
    (t,) = workloads.make_inputs(workloads.CONFIGS["c5_fw_u16"], n_sample)
    t0 = time.perf_counter()
    out = oracle.semiring_close(t, 16, "anti", threads=threads)
    dt = time.perf_counter() - t0
    return n_sample ** 3 / dt, dt, out, t


def cpu_mul_sample(cfg, n_sample: int, threads: int = 0):
    import oracle
    from paper_1705_08743_b200 import workloads
    a, b = workloads.make_inputs(cfg, n_sample)
    t0 = time.perf_counter()
    out = oracle.semiring_mul(a, b, n_sample, cfg.width, "anti", threads=threads)
    dt = time.perf_counter() - t0
    return n_sample ** 3 / dt, dt, out


def cpu_baseline_and_parity(cfg):
    """cpu_baseline (the reference algorithm, C restatement, all host threads,
    on CPU_SAMPLE_N of the same generator) and this GPU's result on the same
    sample compared bit for bit."""
    import oracle
    from paper_1705_08743_b200 import AntidistMatrix, workloads
    oracle.build()
    thr = oracle.max_threads()
    n_s = CPU_SAMPLE_N[cfg.op]
    if cfg.op == "closure":
        cps, cdt, cpu_out, t_in = cpu_fw_sample(n_s, thr)
        gpu_out = AntidistMatrix(n_s, n_s, 16, t_in).transitive_closure().data
    else:
        cps, cdt, cpu_out = cpu_mul_sample(cfg, n_s, thr)
        ai, bi = workloads.make_inputs(cfg, n_s)
        gpu_out = (AntidistMatrix(n_s, n_s, cfg.width, ai) * AntidistMatrix(n_s, n_s, cfg.width, bi)).data
    return {
        "cpu_baseline": {
            "value": cps, "unit": UNIT, "cores": thr, "kind": "port",
            "sample": f"{cfg.name} generator at n={n_s}, one "
                      f"{'closure' if cfg.op == 'closure' else 'product'} "
                      f"({cdt:.2f} s), C restatement of the reference engine, OpenMP rows"},
        "parity": {"n": n_s, "bit_exact_vs_oracle": bool(np.array_equal(gpu_out, cpu_out))},
    }


def run_reference(args, world, rank):
    """--impl reference: the reference algorithm on host cores, same metric."""
    if rank != 0:
        return 0
    import oracle
    from paper_1705_08743_b200 import workloads
    oracle.build()
    cfg = workloads.CONFIGS[args.workload]
    threads = oracle.max_threads()
    # the same sample as cpu_baseline on every run (n fixed); a long --steps /
    # --warmup request is bounded by capping the number of CPU steps instead
    # (~9 s each at n = 8192 on 16 host threads), so the arm ends in ~1 min
    n_sample = CPU_SAMPLE_N[cfg.op]
    steps, warmup = max(1, min(args.steps, REF_MAX_STEPS)), min(args.warmup, REF_MAX_WARMUP)

    def step():
        if cfg.op == "closure":
            return cpu_fw_sample(n_sample, threads)[1]
        if cfg.op == "mul":
            return cpu_mul_sample(cfg, n_sample, threads)[1]
        inputs = workloads.make_inputs(cfg, n_sample)
        t0 = time.perf_counter()
        if cfg.op == "bool_mul":
            oracle.bool_mul(oracle.pack_bits(inputs[0]), oracle.pack_bits(inputs[1]), n_sample, threads)
        else:
            oracle.bool_close(oracle.pack_bits(inputs[0]), threads)
        return time.perf_counter() - t0

    for _ in range(warmup):
        step()
    secs = [step() for _ in range(steps)]
    total = sum(secs)
    value = n_sample ** 3 * steps / total
    sample = (f"{cfg.name} at n={n_sample} (same generator and seed), one "
              f"{'closure' if 'closure' in cfg.op else 'product'} per step")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": steps, "warmup": warmup, "steps_requested": args.steps, "warmup_requested": args.warmup,
        "ms_per_step": total / steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "u16" if cfg.width == 16 else f"u{cfg.width}", "data": "synthetic (seeded generator)",
        "config": {"workload": cfg.name, "n": n_sample, "full_n": cfg.n,
                   "sample": "the cpu_baseline sample of the GPU arm (same n, generator and seed)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "reference = the reference package's numpy engine restated in C (oracle/), "
                "OpenMP over rows; the reference itself is pure Python/numpy (1 core)",
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------- GPU

def run_ours(args, world, rank, local_rank):
    import torch
    import torch.distributed as dist
    from paper_1705_08743_b200 import AntidistMatrix, _native, engines, sharded, workloads

    # SMX_BENCH_BACKEND=gloo: functional check of the multi-rank path with more
    # ranks than GPUs (ranks share a device; gloo's host-side broadcast means no
    # kernel ever waits on another rank).  Timings from such a run mean nothing.
    backend = os.environ.get("SMX_BENCH_BACKEND", "nccl")
    if backend != "nccl":
        local_rank %= torch.cuda.device_count()
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        if backend == "nccl":
            # communicator setup lines (rank, nranks, transport) in the log
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            # NCCL's internal stream at the highest priority: the pivot-panel
            # broadcast is on the critical path of the next round and must not
            # queue behind the bulk GEMM's CTAs (sharded.py, _bcast)
            opts = dist.ProcessGroupNCCL.Options()
            opts.is_high_priority_stream = True
            dist.init_process_group("nccl", device_id=dev, pg_options=opts)
        else:
            dist.init_process_group(backend)
    cfg = workloads.CONFIGS[args.workload]
    n = args.n or cfg.n
    lib = _native.lib()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- inputs (host generation, then HBM) --------------------------------
    if world > 1:   # the sharded closure's block (smx_fw_sharded_block)
        block = lib.smx_fw_sharded_block(n, world, cfg.width // 8)
    else:   # the single-GPU closure's own choice (smx_fw_block_for)
        block = lib.smx_fw_block_for(n, cfg.width // 8)
    if cfg.op == "closure":
        r0, r1 = sharded.row_range(n, world, rank, block) if world > 1 else (0, n)
        (host,) = workloads.make_inputs(cfg, n, rows=(r0, r1))
        src = torch.from_numpy(host).to(dev)
        work = torch.empty_like(src)
        # the C-ABI sharded closure (csrc/sharded.cu): NCCL broadcast on the
        # library's high-priority side stream, or a gloo callback
        fw = sharded.NativeShardedFW(n, rank, world, cfg.width, anti=True, block=block)
        ws_bytes = lib.smx_fw_workspace_bytes(n, src.shape[1], cfg.width // 8)
        ws = _native.workspace(ws_bytes, dev)

        def step():
            work.copy_(src)
            if world == 1:
                _native.check(getattr(lib, f"smx_fw_u{cfg.width}")(
                    work.data_ptr(), n, work.shape[1], _native.SMX_ANTI, ws.data_ptr(), ws_bytes,
                    _native.stream_ptr(dev)), "fw")
            else:
                fw.run(work)
        units_per_step = n ** 3
    elif cfg.op == "mul":
        r0, r1 = sharded.row_range(n, world, rank, 128) if world > 1 else (0, n)
        a_host, b_host = workloads.make_inputs(cfg, n, rows=(r0, r1))
        a, b = torch.from_numpy(a_host).to(dev), torch.from_numpy(b_host).to(dev)
        out = torch.empty((a.shape[0], b.shape[1]), dtype=a.dtype, device=dev)

        def step():
            sharded.sharded_mul(a, b, n, cfg.width, True, out)
        units_per_step = n ** 3
    else:
        raise SystemExit(f"bench workload {cfg.name}: use tools/perf_probe.py for Boolean configs")

    # ---- timed region -------------------------------------------------------
    for _ in range(args.warmup):
        step()
    barrier()
    launches0 = lib.smx_launch_count()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # dominant-kernel trace: CUDA events around every phase-3 launch of the
    # first timed step (FW), or around each product (mul), on its own stream
    rounds = -(-n // block)
    step_events = []
    if cfg.op == "closure":
        # phase-3 (3b at N > 1) launches of the first timed step, CUDA-event timed
        _native.check(lib.smx_fw_trace_arm(rounds), "trace arm")
    with ClockSampler(local_rank) as clocks:
        s.record()
        for i in range(args.steps):
            if cfg.op == "mul":
                ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                ev[0].record()
                step()
                ev[1].record()
                step_events.append(ev)
            else:
                step()
        e.record()
        barrier()
    if cfg.op == "closure" and world > 1:
        sharded_trace = read_fw_trace(lib, rounds)
    launches = lib.smx_launch_count() - launches0
    secs = s.elapsed_time(e) / 1e3
    t = torch.tensor([secs], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    secs = float(t.item())
    value = units_per_step * args.steps / secs

    result = {}
    if world > 1:
        # e2e at N GPUs through the public sharded API: every rank copies its
        # row panel in from pinned host memory, runs the sharded closure /
        # product and copies its result rows back, all inside the timed loop
        if cfg.op == "closure":
            pin_in = torch.from_numpy(host).pin_memory()

            def e2e_step():
                work.copy_(pin_in, non_blocking=True)
                fw.run(work)
                pin_out.copy_(work, non_blocking=True)
            pin_out = torch.empty_like(pin_in).pin_memory()
            h2d, d2h = pin_in.numel() * pin_in.element_size(), pin_out.numel() * pin_out.element_size()
        else:
            pa, pb = torch.from_numpy(a_host).pin_memory(), torch.from_numpy(b_host).pin_memory()
            pin_out = torch.empty((a_host.shape[0], b_host.shape[1]), dtype=pa.dtype).pin_memory()

            def e2e_step():
                a.copy_(pa, non_blocking=True)
                b.copy_(pb, non_blocking=True)
                sharded.sharded_mul(a, b, n, cfg.width, True, out)
                pin_out.copy_(out, non_blocking=True)
            h2d = (pa.numel() + pb.numel()) * pa.element_size()
            d2h = pin_out.numel() * pin_out.element_size()
        for _ in range(3):   # warm-up (see the N = 1 e2e below)
            e2e_step()
        barrier()
        es, ee = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e2e_steps = 2
        es.record()
        for _ in range(e2e_steps):
            e2e_step()
        ee.record()
        barrier()
        te = torch.tensor([es.elapsed_time(ee) / 1e3 / e2e_steps], dtype=torch.float64, device=dev)
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e_secs = float(te.item())
        hb = torch.tensor([h2d, d2h], dtype=torch.float64, device=dev)
        dist.all_reduce(hb)
        result["e2e"] = {"value": units_per_step / e2e_secs, "unit": UNIT,
                         "h2d_bytes_per_step": int(hb[0].item()), "d2h_bytes_per_step": int(hb[1].item()),
                         "ms_per_step": e2e_secs * 1e3, "note": "summed over ranks; max time over ranks"}
        if cfg.op == "closure":
            result["roofline"] = sharded_roofline(sharded_trace, secs / args.steps, n, block, world, dev)
            digest = full_size_digest(cfg.name, n)
            if args.check or (digest is not None and backend == "nccl"):
                result["parity_sharded"] = sharded_parity(work, cfg, n, world, rank, block, dev, digest)

    # ---- parity of this very run at the oracle size (rank 0, N = 1) ------------
    if rank == 0 and world == 1:
        # dominant kernel, timed live in the timed region (trace / events above)
        if cfg.op == "closure":
            import ctypes
            ms_arr = (ctypes.c_float * rounds)()
            cells_arr = (ctypes.c_longlong * rounds)()
            cnt = lib.smx_fw_trace_read(ms_arr, cells_arr, rounds)
            if cnt <= 0:
                raise RuntimeError(f"phase-3 trace read failed ({cnt})")
            dom_secs_total = sum(ms_arr[i] for i in range(cnt)) / 1e3
            dom_cells = sum(cells_arr[i] for i in range(cnt))
            dom_launches = cnt
            step_secs = secs / args.steps
            # per launch: A panel n x B, B panel B x n, C read + written
            alg_bytes = (2 * n * block + 2 * n * n) * cfg.width // 8
        else:
            times = [ev[0].elapsed_time(ev[1]) / 1e3 for ev in step_events]
            dom_secs_total = sum(times)
            dom_cells = n ** 3 * len(times)
            dom_launches = len(times)
            step_secs = secs / args.steps
            alg_bytes = 3 * n * n * cfg.width // 8
        peaks, sms = measure_issue_peak()
        result["peaks"] = peaks
        achieved = dom_cells / dom_secs_total
        # the ceiling is the best issue rate of either mix: one VIADDMNMX.U16x2
        # updates 2 cells, and the VIMNMX + VIADDMNMX pair issues no faster
        issue = max(peaks["one"], peaks["pair"])
        peak_cells = 2.0 * issue            # one u16x2 instruction updates 2 cells at best
        traffic = load_traffic(cfg.name)
        result["roofline"] = {
            "bound": "int_issue", "achieved": achieved / 1e12, "peak": peak_cells / 1e12,
            "unit": "Tcell/s", "frac": achieved / peak_cells, "traffic": traffic,
            "traffic_unit": "DRAM bytes per launch (ncu, profiles/traffic.json)",
            "kernel": ("packed_gemm_u16_kernel (FW phase 3, per round)" if cfg.op == "closure" and cfg.width == 16
                       else "packed_gemm_u16_kernel (product; K-chunk packs included)" if cfg.width == 16
                       else "semiring_gemm_kernel"),
            "sms": sms,
            "issue_rate": issue,
            "launches_timed": dom_launches,
            "avg_launch_ms": dom_secs_total / dom_launches * 1e3,
            "share_of_step": dom_secs_total / dom_launches *
                             (rounds if cfg.op == "closure" else 1) / step_secs,
            "instr_per_cell": issue / achieved if achieved else None,
            "peak_source": (f"measured in this run: smx_int_issue_probe on {sms} SMs issues "
                            f"{issue / 1e12:.2f} T u16x2-instr/s (VIADDMNMX.U16x2 alone; the VIMNMX + "
                            f"VIADDMNMX pair: {peaks['pair'] / 1e12:.2f} T); peak = 2 cell-updates per "
                            f"instruction. The general saturating u16 update needs 2 instr per 2 cells "
                            f"(ceiling 0.5); verified-bounded / certified tiles and u8 need 1"),
            "algorithmic_bytes_per_launch": alg_bytes,
        }
        # the other roof: DRAM bandwidth the dominant kernel draws, against the
        # driver-measured HBM copy bandwidth (MEASURED_PEAKS.json)
        avg_s = dom_secs_total / dom_launches
        hbm = None
        mp = REPO / "MEASURED_PEAKS.json"
        if mp.exists():
            try:
                hbm = float(json.loads(mp.read_text()).get("hbm_gbs"))
            except (ValueError, TypeError):
                hbm = None
        bytes_l = traffic if traffic else alg_bytes
        result["roofline"]["hbm_gbs_achieved"] = bytes_l / avg_s / 1e9
        result["roofline"]["hbm_gbs_peak"] = hbm
        result["roofline"]["hbm_frac"] = (bytes_l / avg_s / 1e9 / hbm) if hbm else None
        # e2e through the public API with host buffers
        if cfg.op == "closure":
            # the reference's own call on an ordinary (pageable) numpy array:
            # AntidistMatrix(n, n, w, host).transitive_closure().data
            # (antidist.py:263-273).  The matrix is host-backed; the closure is
            # one smx_fw_host_u16 call that stages the rows in through
            # page-locked slots and closes them as they arrive, copies finished
            # rows out into page-locked memory while the rest runs, and .data
            # is a view of that memory (as the reference's is of its array)
            def e2e_step():
                return AntidistMatrix(n, n, cfg.width, host).transitive_closure().data
            h2d = d2h = host.nbytes
        else:
            # the reference's own product call on numpy arrays:
            # (AntidistMatrix(n, n, w, a) * AntidistMatrix(n, n, w, b)).data
            # (antidist.py:226-250): the streamed host product (left operand
            # staged in by row groups beside the products, result rows out)
            def e2e_step():
                return (AntidistMatrix(n, n, cfg.width, a_host) * AntidistMatrix(n, n, cfg.width, b_host)).data
            h2d = a_host.nbytes + b_host.nbytes
            d2h = n * b_host.shape[1] * b_host.itemsize
        e2e_steps = 2 if n >= 16384 else 5
        # 3 warm-up calls (the product's public path records one replay graph
        # per buffer layout the caching allocator hands out)
        for _ in range(3):
            e2e_step()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            e2e_step()
        torch.cuda.synchronize()
        e2e_secs = (time.perf_counter() - t0) / e2e_steps
        result["e2e"] = {"value": units_per_step / e2e_secs, "unit": UNIT,
                         "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                         "ms_per_step": e2e_secs * 1e3}
        if cfg.op != "closure":
            result["e2e"]["call"] = ("(AntidistMatrix(n, n, 16, a) * AntidistMatrix(n, n, 16, b)).data "
                                     "(pageable numpy in, page-locked result out)")
        if cfg.op == "closure":
            result["e2e"]["call"] = ("AntidistMatrix(n, n, 16, host_ndarray).transitive_closure().data "
                                     "(pageable numpy in, page-locked result out)")
            # the same closure from a page-locked buffer into a page-locked
            # buffer through the C-ABI's host-buffer entry (no staging)
            pinned = torch.from_numpy(host).pin_memory()
            res_host = torch.empty_like(pinned).pin_memory()

            def pinned_step():
                AntidistMatrix.closure_of_host(pinned, cfg.width, out=res_host)
            pinned_step()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(2):
                pinned_step()
            torch.cuda.synchronize()
            d_secs = (time.perf_counter() - t0) / 2
            result["e2e_pinned"] = {"value": units_per_step / d_secs, "unit": UNIT, "ms_per_step": d_secs * 1e3,
                                    "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                                    "call": "AntidistMatrix.closure_of_host(pinned, 16, out=pinned_out) "
                                            "(smx_fw_host_u16)"}
            del pinned, res_host
        # CPU baseline + parity at the oracle size (same generator)
        if not args.no_cpu:
            result.update(cpu_baseline_and_parity(cfg))
        if not args.no_secondary:
            result["secondary"] = secondary(dev)

    if rank == 0 and world > 1 and not args.no_cpu and backend == "nccl":
        # the same bounded CPU sample at N > 1 (after the timed region; rank 0)
        result.update(cpu_baseline_and_parity(cfg))

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": secs / args.steps * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None,
            "dtype": f"u{cfg.width}", "data": "synthetic (seeded generator, SURVEY 8(d))",
            "config": {"workload": cfg.name, "op": cfg.op, "n": n, "density": cfg.p,
                       "weights": f"U[1,{cfg.wmax}]", "seed": cfg.seed,
                       "parallelism": f"row-panel x{world}" if world > 1 else "single GPU",
                       "l2": "inputs larger than L2 (no flush needed)" if n * n * cfg.width // 8 > 126e6
                       else "inputs fit L2"},
            "gpu_launches": int(launches),
            "clocks": clocks.summary(),
        }
        line.update(result)
        roof = line.get("roofline")
        mhz = line["clocks"].get("sm_mhz") if isinstance(line.get("clocks"), dict) else None
        if roof and mhz:
            # the probe against the nominal packed-integer pipe (64 lanes/clk/SM)
            # at the SM clock held during the timed region
            nominal = 2.0 * roof["sms"] * 64 * mhz * 1e6
            roof["probe_lanes_per_clk_per_sm"] = roof["issue_rate"] / (roof["sms"] * mhz * 1e6)
            roof["nominal_peak"] = nominal / 1e12
            roof["frac_of_nominal"] = roof["achieved"] * 1e12 / nominal
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def secondary(dev):
    """Quick device timings of the other BASELINE configs (full size)."""
    import torch
    from paper_1705_08743_b200 import AntidistMatrix, BoolMatrix, engines, workloads
    out = {}
    for name in ("c3_mul_u8", "c3_mul_u16"):
        cfg = workloads.CONFIGS[name]
        a, b = workloads.make_inputs(cfg)
        ta, tb = torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev)
        res = torch.empty_like(ta)
        t = cuda_time(lambda: engines.lane_mul(ta, tb, cfg.n, cfg.width, True, res), 10, 2)
        out[name] = {"n": cfg.n, "seconds": t, "cells_per_s": cfg.n ** 3 / t}
    cfg = workloads.CONFIGS["c4_fw_u16"]
    (t8k,) = workloads.make_inputs(cfg)
    src = torch.from_numpy(t8k).to(dev)
    w = torch.empty_like(src)

    def fw8k():
        w.copy_(src)
        engines.lane_close_(w, cfg.n, 16, True)
    t = cuda_time(fw8k, 5, 2)   # 2 warm-ups: the second records the replay graph
    out["c4_fw_u16"] = {"n": cfg.n, "seconds": t, "cells_per_s": cfg.n ** 3 / t}
    # the same graph as a DistMatrix (min-plus closure of the complement,
    # antidist.py:331-350) and at u32 lanes (kernels.py:35): same distances
    peaks, _ = measure_issue_peak()
    issue = max(peaks["one"], peaks["pair"])
    ref8k = w.clone()
    dsrc = (65535 - src.to(torch.int32)).to(torch.uint16)
    wd = torch.empty_like(dsrc)

    def fw8k_dist():
        wd.copy_(dsrc)
        engines.lane_close_(wd, cfg.n, 16, False)
    t = cuda_time(fw8k_dist, 5, 2)
    same = bool(torch.equal((65535 - wd.to(torch.int32)).to(torch.uint16), ref8k))
    out["c4_fw_u16_dist"] = {"n": cfg.n, "seconds": t, "cells_per_s": cfg.n ** 3 / t,
                             "frac_of_issue_ceiling": cfg.n ** 3 / t / (2 * issue),
                             "complement_of_anti_closure": same}
    s32 = src.to(torch.int64)
    src32 = torch.where(s32 == 0, torch.zeros_like(s32), s32 + (2 ** 32 - 65536)).to(torch.uint32)
    w32 = torch.empty_like(src32)

    def fw8k_u32():
        w32.copy_(src32)
        engines.lane_close_(w32, cfg.n, 32, True)
    t = cuda_time(fw8k_u32, 3, 2)
    r32 = w32.to(torch.int64)
    back = torch.where(r32 == 0, torch.zeros_like(r32), r32 - (2 ** 32 - 65536))
    out["c4_fw_u32"] = {"n": cfg.n, "seconds": t, "cells_per_s": cfg.n ** 3 / t,
                        "frac_of_issue_ceiling": cfg.n ** 3 / t / issue,
                        "ceiling_note": "u32: 1 cell per instruction at best (VIADDMNMX on bounded tiles)",
                        "same_distances_as_u16": bool(torch.equal(back.to(torch.int32),
                                                                  ref8k.to(torch.int32)))}
    out["c4_fw_u16"]["frac_of_issue_ceiling"] = out["c4_fw_u16"]["cells_per_s"] / (2 * issue)
    del ref8k, dsrc, wd, s32, src32, w32, r32, back
    cfg = workloads.CONFIGS["c1_bool_mul"]
    a, b = workloads.make_inputs(cfg)
    ma, mb = BoolMatrix.from_numpy(a), BoolMatrix.from_numpy(b)
    for eng in ("bool_mul_tc", "bool_mul_bits"):
        fn = getattr(engines, eng)
        t = cuda_time(lambda: fn(ma, mb), 50, 5)
        out[f"c1_{eng}"] = {"n": cfg.n, "seconds": t, "cells_per_s": cfg.n ** 3 / t,
                            "note": "public BoolMatrix call incl. unpack/alloc/Python"}
    # the tensor-core kernel alone (C1 shape and a throughput shape) against
    # the measured dense int8 peak (cuBLAS torch._int_mm, 8192^3)
    from paper_1705_08743_b200 import _native
    lib = _native.lib()
    a8 = torch.randint(-127, 127, (8192, 8192), dtype=torch.int8, device=dev)
    t = cuda_time(lambda: torch._int_mm(a8, a8.t()), 10, 2)
    int8_peak = 2 * 8192 ** 3 / t
    del a8
    tc = {"int8_peak_ops_per_s": int8_peak, "peak_source": "measured: torch._int_mm 8192^3 (cuBLAS)"}
    for n_tc in (1024, 2048, 4096, 8192):
        A = (torch.rand((n_tc, n_tc), device=dev) < 0.05).to(torch.uint8)
        Bt = (torch.rand((n_tc, n_tc), device=dev) < 0.05).to(torch.uint8)
        # the same 0/1 operands as E2M1 nibbles (1.0 = 0b0010), two per byte
        A4 = (A[:, 0::2] * 2 + A[:, 1::2] * 32).contiguous()
        Bt4 = (Bt[:, 0::2] * 2 + Bt[:, 1::2] * 32).contiguous()
        o = torch.zeros((n_tc, n_tc // 32), dtype=torch.int32, device=dev)
        o4 = torch.zeros_like(o)
        f8 = lambda: _native.check(lib.smx_bool_gemm_i8(  # noqa: E731
            A.data_ptr(), Bt.data_ptr(), None, o.data_ptr(), n_tc, n_tc, n_tc, n_tc, n_tc, n_tc // 32, 0,
            _native.stream_ptr(dev)), "tc")
        f4 = lambda: _native.check(lib.smx_bool_gemm_f4(  # noqa: E731
            A4.data_ptr(), Bt4.data_ptr(), o4.data_ptr(), n_tc, n_tc, n_tc, n_tc // 2, n_tc // 2, n_tc // 32, 0,
            _native.stream_ptr(dev)), "tc f4")
        te = cuda_time(f4, 20 if n_tc <= 4096 else 5, 2)
        # device rate: back-to-back launches in one graph (an eager Python
        # loop of launches is host-bound at this size: ~5 us per launch)
        it, reps = (20, 20) if n_tc <= 4096 else (3, 2)
        t8 = graph_time(f8, it, reps)
        t = graph_time(f4, it, reps)
        tc[f"n{n_tc}"] = {"kernel_us": t * 1e6, "ops_per_s": 2 * n_tc ** 3 / t,
                          "frac_of_int8_peak": 2 * n_tc ** 3 / t / int8_peak,
                          "eager_launch_us": te * 1e6,
                          "i8_kernel_us": t8 * 1e6, "i8_frac_of_int8_peak": 2 * n_tc ** 3 / t8 / int8_peak,
                          "same_bits_as_i8": bool(torch.equal(o, o4))}
    # C1-shaped products many per launch (bool_mul_many on 128-multiple
    # shapes): the batched kernel, three CTAs per SM
    nb = 16
    A = (torch.rand((nb * 1024, 1024), device=dev) < 0.05).to(torch.uint8)
    Bt = (torch.rand((nb * 1024, 1024), device=dev) < 0.05).to(torch.uint8)
    A4 = (A[:, 0::2] * 2 + A[:, 1::2] * 32).contiguous()
    Bt4 = (Bt[:, 0::2] * 2 + Bt[:, 1::2] * 32).contiguous()
    o = torch.zeros((nb * 1024, 32), dtype=torch.int32, device=dev)
    o4 = torch.zeros_like(o)
    f8 = lambda: _native.check(lib.smx_bool_gemm_i8_batched(  # noqa: E731
        A.data_ptr(), Bt.data_ptr(), o.data_ptr(), nb, 1024, 1024, 1024, 1024, 1024, 32, 0,
        _native.stream_ptr(dev)), "tc batched")
    f4 = lambda: _native.check(lib.smx_bool_gemm_f4_batched(  # noqa: E731
        A4.data_ptr(), Bt4.data_ptr(), o4.data_ptr(), nb, 1024, 1024, 1024, 512, 512, 32, 0,
        _native.stream_ptr(dev)), "tc f4 batched")
    t8 = graph_time(f8, 10, 10) / nb
    t = graph_time(f4, 10, 10) / nb
    tc["n1024_batch16"] = {"kernel_us_per_product": t * 1e6, "ops_per_s": 2 * 1024 ** 3 / t,
                           "frac_of_int8_peak": 2 * 1024 ** 3 / t / int8_peak,
                           "i8_kernel_us_per_product": t8 * 1e6,
                           "i8_frac_of_int8_peak": 2 * 1024 ** 3 / t8 / int8_peak,
                           "same_bits_as_i8": bool(torch.equal(o, o4)),
                           "note": "16 independent 1024^3 products per launch (smx_bool_gemm_f4_batched)"}
    del A, Bt, A4, Bt4, o, o4
    tc["kernel"] = ("E2M1 nibble operands, tcgen05 kind::mxf4 with unit scale factors (smx_bool_gemm_f4, the "
                    "default of the public product): bool_f4 split-K CTA pair at 1024, the plain kernel above; "
                    "i8_* = the same product on byte operands, kind::i8 (smx_bool_gemm_i8); kernel_us = device "
                    "time per launch, back-to-back launches replayed from one CUDA graph; the denominator is "
                    "the dense int8 peak (cuBLAS), which the nibble kernels may exceed")
    out["bool_tc_gemm_kernel"] = tc
    cfg = workloads.CONFIGS["c2_bool_warshall"]
    (t2,) = workloads.make_inputs(cfg)
    m2 = BoolMatrix.from_numpy(t2)
    for eng in ("bool_closure_tc", "bool_closure_bits"):
        fn = getattr(engines, eng)
        t = cuda_time(lambda: fn(m2), 10, 2)
        out[f"c2_{eng}"] = {"n": cfg.n, "seconds": t, "cells_per_s": cfg.n ** 3 / t,
                            "frac_of_int8_tc_peak": 2 * cfg.n ** 3 / t / int8_peak}
    # entrywise ops at C5 size, HBM-bound (one 16-byte packed
    # SIMD pass), against the driver-measured HBM copy bandwidth
    hbm = None
    mp = REPO / "MEASURED_PEAKS.json"
    if mp.exists():
        try:
            hbm = float(json.loads(mp.read_text()).get("hbm_gbs"))
        except (TypeError, ValueError):
            hbm = None
    ne = 32768
    ea = torch.randint(0, 65535, (ne, ne), dtype=torch.int32, device=dev).to(torch.uint16)
    eb = torch.randint(0, 65535, (ne, ne), dtype=torch.int32, device=dev).to(torch.uint16)
    ec = torch.empty_like(ea)
    t = cuda_time(lambda: _native.check(lib.smx_lane_entrywise(
        ea.data_ptr(), eb.data_ptr(), ec.data_ptr(), ne, ne, ne, 2, 1, 0, _native.stream_ptr(dev)), "|"), 10, 2)
    gbs = 3 * ea.numel() * 2 / t / 1e9
    out["entrywise_or_u16"] = {"n": ne, "seconds": t, "gbs": gbs, "hbm_gbs_peak": hbm,
                               "frac_of_hbm": gbs / hbm if hbm else None,
                               "op": "AntidistMatrix | (lanewise max, antidist.py:128-156), 3 x 2 GiB per call"}
    del ea, eb, ec
    # the bit path's own ceiling: one LOP3.LUT (OR of AND on a 32-bit word)
    # per 32 cell-updates at the measured LOP3 issue rate
    bits = out["c2_bool_closure_bits"]
    bits["bit_alu_ceiling_cells_per_s"] = 32 * peaks["lop3"]
    bits["frac_of_bit_alu_ceiling"] = bits["cells_per_s"] / (32 * peaks["lop3"])
    bits["lop3_issue_per_s"] = peaks["lop3"]
    return out


def relaunch_under_torchrun(args) -> int:
    """`bench.py --gpus N` (N > 1) started as a plain process: re-run this
    command as N ranks under torch.distributed.run (127.0.0.1, a free port),
    the layout the driver uses; rank 0 prints the line."""
    import socket
    import subprocess
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve()),
           *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch_under_torchrun(args)
    world, rank, local = dist_env()
    if "WORLD_SIZE" in os.environ and world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        return run_reference(args, world, rank)
    return run_ours(args, world, rank, local)


if __name__ == "__main__":
    sys.exit(main())
