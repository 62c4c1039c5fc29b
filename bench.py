"""Benchmark of the fused ternary widely-linear GEMV (FairyFuse, arXiv 2604.20913) on B200.

Default workload (BASELINE.json config 4, the 7B decode linear stack): one step = one token
through 32 decoder layers x 7 widely-linear projections (q,k,v,o 2048->2048; gate,up
2048->5504; down 5504->2048, complex), B = 1, launched as 4 stages per layer (q/k/v and
gate/up share their input, so each group is one launch), every stage's output rows sharded
over the GPUs and all-gathered (NCCL).  The 1.62 GB of packed weights per step is > 12x L2, so
every step streams its weights from HBM (no flush needed).

    python bench.py [--gpus N --steps K --warmup W] [--workload c4|c2|c3a|c3b|c5] [--batch B]
    python bench.py --impl reference ...    # the C fp64 oracle on the host cores

Prints ONE JSON line on rank 0 (contract in the task statement; fields documented in
DESIGN.md §8).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "WL-GEMV packed-weight HBM GB/s (% of B200 peak), us/layer at 7B shapes"
L2_BYTES = 126 * 2**20


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 100 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_id: str):
        self.gpu_id, self.rows, self.proc, self.thread = gpu_id, [], None, None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", self.gpu_id, f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def stop(self):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()
        if self.thread is not None:
            self.thread.join(timeout=2)

    def summary(self, peaks):
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if r[2 + i].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else peaks.get("sm_max_mhz"),
                "reasons": reasons, "samples": len(self.rows)}


# --------------------------------------------------------------------------- distributed
def _dist_init(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def _gpu_id(local):
    import torch
    try:
        u = str(torch.cuda.get_device_properties(local).uuid)
        return u if u.startswith("GPU-") else "GPU-" + u
    except Exception:
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        return vis.split(",")[local] if vis else str(local)


# --------------------------------------------------------------------------- oracle (CPU)
def oracle_sample(layers=(0,), seed=0, rows=None):
    """Generate (host, untimed) the planar inputs of the listed decoder layers' 7 projections."""
    import oracle as orc
    import ww_inputs as wi
    work = []
    for l in layers:
        for p, spec in enumerate(wi.C4_PROJS):
            s = wi.layer_seed(seed, l, p)
            nr = spec.n if rows is None else min(rows, spec.n)
            planes = wi.planes(s, spec.n, spec.m, spec.dist, 0, nr)
            sc = wi.scales(s, spec.n, True, spec.scale_lo, spec.scale_hi)[:nr]
            x = wi.activations(s, spec.m, 1)
            work.append((orc.pack_planar(planes), nr, spec.m, np.ascontiguousarray(sc), x))
    return work


def oracle_time(work, omp=False):
    """One pass of the C fp64 oracle over the sample, in its two phases:
    (a) unpack + build the dense complex rows, (b) evaluate Eq. 1.  Returns
    (unpack_s, eval_s, packed_bytes)."""
    import oracle as orc
    tu = te = 0.0
    nbytes = 0
    for planar, nr, m, sc, x in work:
        t0 = time.perf_counter()
        U, Wd = orc.build_dense(planar, nr, m, sc, omp=omp)
        t1 = time.perf_counter()
        orc.eval_dense(U, Wd, x, orc.CONV_EQ1, omp=omp)
        t2 = time.perf_counter()
        del U, Wd
        tu += t1 - t0
        te += t2 - t1
        nbytes += 16 * nr * ((m + 15) // 16)
    return tu, te, nbytes


def host_info() -> dict:
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        usable = len(os.sched_getaffinity(0))
    except AttributeError:
        usable = os.cpu_count()
    return {"cpu_model": model, "nproc": usable, "cpu_count": os.cpu_count()}


SAMPLE = ("decoder layer 0 of config 4 (q,k,v,o 2048x2048; gate,up 5504x2048; down 2048x5504), "
          "all rows, B=1, EQ1: the C fp64 oracle's unpack + dense build, then direct evaluation")


def cpu_baseline(seed=0, runs=3) -> dict:
    """The oracle as it stands on this host's cores (rank 0, N = 1): median of `runs` passes
    over decoder layer 0, single-threaded and with OpenMP over rows on every usable core,
    unpack timed apart from evaluate.  GB/s of packed weights."""
    import oracle as orc
    work = oracle_sample(layers=(0,), seed=seed)
    out = {}
    for omp in (False, True):
        ts = [oracle_time(work, omp) for _ in range(runs)]
        tu = float(np.median([t[0] for t in ts]))
        te = float(np.median([t[1] for t in ts]))
        tt = float(np.median([t[0] + t[1] for t in ts]))
        nb = ts[0][2]
        out["omp" if omp else "single"] = {
            "value": round(nb / tt / 1e9, 6), "cores": orc.num_threads(omp),
            "unpack_s": round(tu, 4), "eval_s": round(te, 4), "total_s": round(tt, 4)}
    allc = out["omp"]
    return {"value": allc["value"], "unit": "GB/s", "cores": allc["cores"], "kind": "oracle",
            "sample": SAMPLE + f"; median of {runs} runs; value = OpenMP over rows on all "
                      "usable cores (`single` = one thread)",
            "single_thread": out["single"], "all_cores": allc,
            "paper_alg1_avx512": alg1_baseline(work, runs), **host_info()}


def alg1_baseline(work, runs=3) -> dict:
    """The paper's own CPU kernel (Algorithm 1, AVX-512F + BMI2, OpenMP rows; NEXT-4) on the
    same sample: a like-for-like CPU datapath beside the oracle.  GB/s of packed weights."""
    try:
        import cpu_alg1
        if not cpu_alg1.supported():
            return {"unavailable": "host CPU lacks AVX-512F or BMI2"}
    except OSError as e:
        return {"unavailable": f"libww_cpu.so: {e}"}
    out = {}
    for name, T in (("single", 1), ("all_cores", 0)):
        ts = []
        for _ in range(runs + 1):  # first pass warms the pages
            t0 = time.perf_counter()
            nb = 0
            for planar, nr, m, sc, x in work:
                cpu_alg1.wl_gemv(planar, nr, m, sc, x, 0, T)
                nb += 16 * nr * ((m + 15) // 16)
            ts.append(time.perf_counter() - t0)
        t = float(np.median(ts[1:]))
        out[name] = {"value": round(nb / t / 1e9, 4), "unit": "GB/s", "ms_per_layer": round(1e3 * t, 3),
                     "cores": 1 if T == 1 else cpu_alg1.max_threads()}
    return out


def run_reference(args, world, rank):
    """--impl reference: the C fp64 oracle as it stands, on the host cores (rank 0 only), OpenMP
    over rows on every usable core; one step = decoder layer 0 of config 4."""
    if rank != 0:
        return
    import oracle as orc
    work = oracle_sample(layers=(0,), seed=args.seed)
    for _ in range(args.warmup):
        oracle_time(work, omp=True)
    ts, nb = [], 0
    for _ in range(args.steps):
        tu, te, nb = oracle_time(work, omp=True)
        ts.append(tu + te)
    t = float(np.sum(ts))
    value = nb * args.steps / t / 1e9
    cores = orc.num_threads(True)
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(value, 6), "unit": "GB/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * t / args.steps, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "c4_llama2_7b_wl_decode_stack (oracle sample)", "batch": 1,
                   "sample": SAMPLE},
        "cpu_baseline": {"value": round(value, 6), "unit": "GB/s", "cores": cores,
                         "kind": "oracle", "sample": SAMPLE + "; OpenMP over rows",
                         **host_info()},
        "e2e": {"value": round(value, 6), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }), flush=True)


# --------------------------------------------------------------------------- GPU arm
def run_ours(args, world, rank, local):
    import torch
    import torch.distributed as dist

    import paper_2604_20913_b200 as ww
    from paper_2604_20913_b200.stack import WLStack
    import ww_inputs as wi

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    peaks, peak_kind = _peaks()
    group = dist.group.WORLD if world > 1 else None

    if args.workload == "c4":
        gam = None
        if args.chain == "block":
            from paper_2604_20913_b200.stack import block_gammas
            gam = [tuple(torch.from_numpy(g).to(dev) for g in pair)
                   for pair in block_gammas(args.seed, args.layers, 2048)]
        base = WLStack(layers=args.layers, seed=args.seed, B=args.batch, rank=rank, world=world,
                       pdl=not args.no_pdl, device=dev, group=group, fuse=not args.no_fuse,
                       chain=args.chain if args.engine == "pdl" else "plain", gammas=gam,
                       symm=args.engine == "program" and world > 1, lut_stages=_lut_stages(args))
        if args.engine == "program":
            stack = ProgramRunner(base, args.chain, gam)
        else:
            stack = base
        units = [stack]
        layers_per_step = 7 * args.layers  # widely-linear projections per token
        if args.engine == "program":
            workload = (f"c4_llama2_7b_wl_decode_stack ({args.layers} layers x 7 projections, "
                        "one persistent program launch per token: 4 stages per layer, "
                        + ("each stage's own seeded x, stage i+1 waits for stage i"
                           if args.chain == "plain" else
                           "NEXT-3 decode blocks chained (RMSNorm, identity attention, "
                           "residuals, SiLU(gate)*up fused)") + ")")
        else:
            workload = (f"c4_llama2_7b_wl_decode_stack ({args.layers} layers x 7 projections, "
                        + ("q/k/v and gate/up launched together per shared input: 4 launches "
                           "per layer" if not args.no_fuse else "one launch per projection")
                        + ")")
    else:
        # single-layer configs: R replicas of the layer (>= 4x L2) cycled inside a step
        spec = {"c2": wi.C2, "c3a": wi.C3A, "c3b": wi.C3B, "c5": wi.C3B, "c1": wi.C1}[args.workload]
        stack = _ReplicaLayer(spec, args, rank, world, dev, group)
        units = [stack]
        layers_per_step = stack.R
        workload = f"{spec.name} x {stack.R} rotating replicas (>= 4x L2)"

    s = torch.cuda.Stream(dev)
    if args.x_l2_persist:  # the step's activations stay in L2 while the weights stream past
        ww.keep_in_l2(stack.inputs(), s)
    launches_per_step = 0
    with torch.cuda.stream(s):
        for _ in range(max(args.warmup, 3)):
            launches_per_step = stack.step(s)
    torch.cuda.synchronize(dev)

    graph = None
    if not args.no_graph:
        try:
            with torch.cuda.stream(s):
                stack.step(s)  # one more eager step right before capture
            torch.cuda.synchronize(dev)
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=s):
                stack.step(s)
            with torch.cuda.stream(s):
                for _ in range(2):
                    graph.replay()
            torch.cuda.synchronize(dev)
        except Exception as e:  # NCCL capture unsupported -> eager steps
            graph = None
            if rank == 0:
                print(f"# graph capture failed ({e!r}); timing eager steps", file=sys.stderr)
            torch.cuda.synchronize(dev)

    def one_step():
        if graph is not None:
            graph.replay()
        else:
            stack.step(s)

    # ---------------- timed region: device time, barrier + sync on both sides, max over ranks
    clocks = ClockSampler(_gpu_id(local))
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    clocks.start()
    time.sleep(0.15)
    with torch.cuda.stream(s):
        e0.record(s)
        for _ in range(args.steps):
            one_step()
        e1.record(s)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    clocks.stop()
    ms = e0.elapsed_time(e1)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    ms_step = ms / args.steps

    # whole-job algorithmic bytes per step (sum over ranks)
    alg = torch.tensor([stack.algorithmic_bytes(), stack.packed_act_bytes(), stack.adds()],
                       dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(alg)
    alg_bytes, pa_bytes, adds = (float(v) for v in alg.tolist())
    value = alg_bytes / (ms_step * 1e-3) / 1e9

    # ---------------- per-shape kernel time: a CUDA graph of the same projection of every
    # layer (distinct weights, so HBM-cold), CUDA events on the launching stream
    per_shape = {}
    allgather_us = {}
    kern_ms_total = 0.0
    if args.workload == "c4" and args.engine == "pdl":
        kinds = {}
        for i, st in enumerate(stack.stages):
            kinds.setdefault(st.name, []).append(i)
        for name, idx in kinds.items():
            st0 = stack.stages[idx[0]]
            label = f"{name} {st0.ylocal}x{st0.m}"
            try:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.stream(s):
                    for i in idx:
                        stack.launch(i, s)
                torch.cuda.synchronize(dev)
                with torch.cuda.graph(g, stream=s):
                    for i in idx:
                        stack.launch(i, s)
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                with torch.cuda.stream(s):
                    g.replay()
                    a.record(s)
                    for _ in range(5):
                        g.replay()
                    b.record(s)
                torch.cuda.synchronize(dev)
                per_shape[label] = round(a.elapsed_time(b) * 1e3 / (5 * len(idx)), 3)
                kern_ms_total += per_shape[label] * 1e-3 * len(idx)
            except Exception as e:  # pragma: no cover
                per_shape[label] = f"unavailable: {e!r}"
            if world > 1:  # the same stages' all-gathers alone (SURVEY §8e breakdown)
                try:
                    allgather_us[label] = _time_allgathers(stack, idx, s, dev)
                except Exception as e:  # pragma: no cover - multi-GPU only
                    allgather_us[label] = f"unavailable: {e!r}"

    # ---------------- e2e: host activations in, result out, through the same API calls
    e2e = _e2e(stack, args, s, dev, graph, world, alg_bytes)

    # ---------------- roofline of the dominant kernel (wl_gemv_kernel: every launch)
    # at N=1 the timed step is nothing but WL-GEMV launches, so the kernel's average launch
    # duration is step time / launches; at N>1 the eager per-launch events are used
    launches = max(launches_per_step, 1)
    if world == 1:
        kern_ms_step = ms_step
    else:
        kern_ms_step = kern_ms_total if kern_ms_total > 0 else ms_step
    per_launch_s = kern_ms_step * 1e-3 / launches
    clk = clocks.summary(peaks)
    sm_mhz = peaks.get("sm_max_mhz", 1965.0)
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count
    alu_peak = 128 * nsm * sm_mhz * 1e6 / 1e12  # fp32 add lanes x SMs x max clock, T add/s
    rank_adds = stack.adds()
    achieved_alu = rank_adds / launches / per_launch_s / 1e12
    rank_pa = stack.packed_act_bytes()
    hbm_achieved = rank_pa / launches / per_launch_s / 1e9
    if getattr(stack, "tc", False):  # tcgen05 kind::i8: MACs of the padded contraction
        # MACs of the padded contraction: 4 planes x rows x (m padded to 256) x N columns, N = 3 limbs
        # x (16 or 32) (vector, component) columns (ww_tc.cu)
        kpad = -(-stack.spec.m // 256) * 256
        ncol = 3 * (16 if 2 * stack.B <= 16 else 32)
        macs = stack.R * 4 * stack.nloc * kpad * ncol
        tops = 2 * macs / launches / per_launch_s / 1e12
        i8_peak = 2 * peaks.get("bf16_tflops", 1622.9)  # int8 = 2x the measured bf16 rate
        tc_roof = {"bound": "tensor", "achieved": round(tops, 2), "peak": round(i8_peak, 1),
                   "unit": "TOPS (int8)", "frac": round(tops / i8_peak, 4),
                   "kernel": "wl_tc_kernel (tcgen05.mma kind::i8)",
                   "peak_basis": "measured bf16 TFLOP/s x 2 (int8 nominal ratio)"}
    roof = {"bound": "alu", "achieved": round(achieved_alu, 4), "peak": round(alu_peak, 4),
            "unit": "Tadd/s", "frac": round(achieved_alu / alu_peak, 4),
            "traffic": _ncu_traffic(lut=bool(getattr(stack, "lut_stages", None))),
            "kernel": ("wl_program_kernel (whole step)" if args.engine == "program"
                       and args.workload == "c4" else
                       "wl_lut_kernel" if getattr(stack, "lut_stages", None) else "wl_gemv_kernel<1>"),
            "peak_basis": f"128 fp32 add lanes/clk/SM x {nsm} SMs x {sm_mhz:.0f} MHz (DESIGN.md §8)"
                          + ("; achieved = the 8nm algorithmic adds per launch (the lookup path issues one "
                             "FADD2 per 4 codes and is bound by LDS.64 issue, 64 codes/clk/SM)"
                             if getattr(stack, "lut_stages", None) else ""),
            "hbm": {"achieved": round(hbm_achieved, 1), "peak": peaks.get("hbm_gbs"),
                    "unit": "GB/s", "frac": round(hbm_achieved / peaks.get("hbm_gbs", 6650.0), 4),
                    "peak_kind": peak_kind, "bytes": "packed weights + x per launch"}}

    if rank != 0:
        return
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args.seed)
    out = {
        "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
        "higher_is_better": True, "scaling": "strong" if args.workload == "c4" else "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": workload, "batch": args.batch, "layers_per_step": layers_per_step,
                   "parallelism": f"rows/{world} + NCCL all-gather" if world > 1 else "1 GPU",
                   "graph": graph is not None, "pdl": not args.no_pdl,
                   "nccl_in_graph": bool(graph is not None and world > 1),
                   "x_l2_persist": bool(args.x_l2_persist),
                   "path": ("tcgen05 kind::i8 (wl_tc_kernel)" if getattr(stack, "tc", False)
                            else "predicated FADD2 (wl_gemv_kernel)"
                            + ("; subset-sum lookup (wl_lut_kernel, WW_LAYOUT_LUT81) on stages "
                               + ",".join(sorted(getattr(stack, "lut_stages", ())))
                               if getattr(stack, "lut_stages", None) else "")),
                   "l2": "inputs > L2: 1.62 GB of weights per step streamed from HBM"
                         if args.workload == "c4" else "rotating replicas >= 4x L2",
                   "launch": _launch_configs(ww, stack, args)},
        "us_per_layer": round(1e3 * ms_step / layers_per_step, 3),
        "launches_per_step": launches_per_step,
        "per_shape_us": per_shape,
        "per_shape_allgather_us": allgather_us if world > 1 else None,
        "pct_of_hbm_peak": round(100 * (pa_bytes / (ms_step * 1e-3) / 1e9) / world
                                 / peaks.get("hbm_gbs", 6650.0), 2),
        "hbm_frac": roof["hbm"]["frac"],
        # the FP32-add ALU fraction describes the CUDA-core kernel; on the tensor-core path
        # the adds run in the MMAs (roofline = the int8 tensor rate)
        "alu_frac": None if getattr(stack, "tc", False) else roof["frac"],
        "roofline": tc_roof if getattr(stack, "tc", False) else roof,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clk,
    }
    print(json.dumps(out), flush=True)


def _time_allgathers(stack, idx, s, dev, reps=5):
    """us per all-gather of the listed stages alone (NCCL, in a CUDA graph when capture works,
    else eager), CUDA events on the launching stream, max over ranks."""
    import torch
    import torch.distributed as dist

    def run():
        for i in idx:
            stack.exchange(i)
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    g = None
    try:
        with torch.cuda.stream(s):
            run()
        torch.cuda.synchronize(dev)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            run()
    except Exception:
        g = None
        torch.cuda.synchronize(dev)
    dist.barrier()
    with torch.cuda.stream(s):
        a.record(s)
        for _ in range(reps):
            g.replay() if g is not None else run()
        b.record(s)
    torch.cuda.synchronize(dev)
    t = torch.tensor([a.elapsed_time(b) * 1e3 / (reps * len(idx))], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return {"us": round(float(t.item()), 3), "graph": g is not None}


def _ncu_traffic(lut=False):
    """dram bytes per launch of the dominant kernel from the committed ncu capture, if any."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            t = json.load(f)
            return (t.get("lut") or {}).get("dram_bytes_per_launch") if lut else t.get("dram_bytes_per_launch")
    except Exception:
        return None


def _e2e(stack, args, s, dev, graph, world, alg_bytes):
    """Same metric with host<->device copies in the timed region: pinned host activations
    -> HBM each step, the last projection's gathered output -> host each step.  With a CUDA
    graph over a stack whose launches read stack.X, the inputs are double-buffered: a second
    graph reads the second buffer, and step k's host->device copy runs on a copy stream while
    step k-1 computes (every step still copies its own inputs inside the timed region)."""
    import torch
    import torch.distributed as dist
    import paper_2604_20913_b200 as ww
    from paper_2604_20913_b200.stack import WLStack
    xflat = stack.inputs().view(-1)
    xh = torch.empty(xflat.numel(), dtype=torch.complex64).pin_memory()
    xh.copy_(xflat.cpu())
    last = stack.Y[-1]
    yh = torch.empty(last.numel(), dtype=torch.complex64).pin_memory()
    steps = max(2, args.steps)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    pipelined = graph is not None and isinstance(stack, WLStack)
    if pipelined:
        # both input buffers in one allocation, so one L2 access-policy window (and one
        # persisting carve-out) covers the two graphs' activations
        XA = stack.X
        Xpair = torch.empty((2, XA.numel()), dtype=XA.dtype, device=dev)
        Xpair[0].copy_(XA)
        Xpair[1].copy_(XA)
        gs = []
        try:
            if args.x_l2_persist:
                ww.keep_in_l2(Xpair, s)
            for h in range(2):
                stack.X = Xpair[h]
                with torch.cuda.stream(s):
                    stack.step(s)
                torch.cuda.synchronize(dev)
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=s):
                    stack.step(s)
                gs.append(g)
        finally:
            stack.X = XA
        xins = [Xpair[h].view(-1)[:xflat.numel()] for h in range(2)]  # the same slice of either
        graphs = gs
        cs = torch.cuda.Stream(dev)
        copied = [torch.cuda.Event(), torch.cuda.Event()]
        consumed = [torch.cuda.Event(), torch.cuda.Event()]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    with torch.cuda.stream(s):
        e0.record(s)
        if pipelined:
            cs.wait_event(e0)
        for k in range(steps):
            if pipelined:
                i = k & 1
                with torch.cuda.stream(cs):
                    if k >= 2:
                        cs.wait_event(consumed[i])  # step k-2 has finished reading this buffer
                    xins[i].copy_(xh, non_blocking=True)
                    copied[i].record(cs)
                s.wait_event(copied[i])
                graphs[i].replay()
                consumed[i].record(s)
            else:
                xflat.copy_(xh, non_blocking=True)
                if graph is not None:
                    graph.replay()
                else:
                    stack.step(s)
            yh.copy_(last, non_blocking=True)
        e1.record(s)
    torch.cuda.synchronize(dev)
    if pipelined and args.x_l2_persist:
        ww.keep_in_l2(stack.inputs(), s)
    ms = e0.elapsed_time(e1) / steps
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    return {"value": round(alg_bytes / (ms * 1e-3) / 1e9, 2), "unit": "GB/s",
            "h2d_bytes_per_step": int(xh.numel() * 8), "d2h_bytes_per_step": int(yh.numel() * 8),
            "ms_per_step": round(ms, 4),
            "overlap": ("inputs double-buffered: step k's host->device copy on a copy stream "
                        "during step k-1" if pipelined else "serial copies on the compute stream")}


def _lut_stages(args):
    """Stages of the config-4 stack that run on the lookup path (B = 1, PDL engine, plain chain)."""
    if (args.workload != "c4" or args.engine != "pdl" or args.chain != "plain" or args.batch != 1
            or args.no_fuse or args.lut_stages == "none"):
        return ()
    if args.lut_stages == "auto":
        return ("qkv", "o", "gateup", "down")
    return tuple(x for x in args.lut_stages.split(",") if x)


def _launch_configs(ww, stack, args):
    """ww_query_launch of every distinct launch shape of the step (per-rank rows)."""
    if args.workload == "c4":
        shapes = {}
        for st in stack.stages:
            shapes.setdefault(f"{st.name} {st.ylocal}x{st.m}", (st.ylocal, st.m))
    else:
        shapes = {f"{stack.spec.name} {stack.nloc}x{stack.spec.m}": (stack.nloc, stack.spec.m)}
    if getattr(stack, "tc", False):
        return {k: {"kernels": "tc_limbs_kernel (2B+1 CTAs x 1024 threads) + wl_tc_kernel (544 threads, "
                               "one CTA per 32-row tile; the K range split over a thread-block cluster of "
                               "up to 4 CTAs when tiles < SMs and B <= 8)",
                    "tiles": -(-n // 32)} for k, (n, m) in shapes.items()}
    out = {k: ww.query_launch(ww.Layer(max(n, 1), m), args.batch) for k, (n, m) in shapes.items()}
    for k, (n, m) in shapes.items():  # lookup stages: wl_lut_kernel's launch shape (ww_lut.cu)
        if k.split()[0] in getattr(stack, "lut_stages", ()):
            steps = -(-m // 512)
            cl = -(-steps // 2)
            out[k] = {"kernel": "wl_lut_kernel", "block": 512, "smem_bytes": 231424, "cluster": cl,
                      "grid": f"min(#SMs // {cl}, resident clusters) x {cl}", "steps_of_512_columns": steps,
                      "columns_per_cta": 1024}
    return out


class ProgramRunner:
    """The C4 stack as ONE persistent program launch per token (ww_program_run): the same
    weights, scales and gathered outputs as the per-launch WLStack."""

    def __init__(self, base, chain, gam):
        import paper_2604_20913_b200 as ww
        from paper_2604_20913_b200.stack import program_stages
        self.base, self.chain, self.gam = base, chain, gam
        if base.world == 1:
            self.prog = ww.Program([program_stages(base, [base], chain, gam)], world=1)
        else:  # one rank per GPU: outputs and sync words in symmetric memory (NEXT-1)
            self.prog = ww.Program([program_stages(base, None, chain, gam)], world=base.world,
                                   rank_base=base.rank, sync=base.symm.sync_ptrs())
        self.stages, self.X, self.Y = base.stages, base.X, base.Y

    def step(self, stream=None):
        self.prog.run(stream)
        return 1

    def inputs(self):
        return self.base.X if self.chain == "plain" else self.base.X[:self.base.stages[0].m]

    def algorithmic_bytes(self):
        return self.base.algorithmic_bytes()

    def packed_act_bytes(self):
        return self.base.packed_act_bytes()

    def adds(self):
        return self.base.adds()


class _ReplicaLayer:
    """A single BASELINE layer shape with R rotating weight replicas (>= 4x L2 in total),
    one step = one launch per replica; row-sharded like the stack when world > 1."""

    def __init__(self, spec, args, rank, world, dev, group):
        import torch
        import paper_2604_20913_b200 as ww
        import ww_inputs as wi
        self.ww, self.spec, self.rank, self.world, self.group = ww, spec, rank, world, group
        self.B = args.batch
        sh = ww.shard_plan(spec.n, spec.m, world, rank)
        self.shard, self.nloc = sh, sh.row_end - sh.row_begin
        # batches of >= 4 vectors run on the tensor cores (ww_wl_gemv_batched_tc, weights in
        # WW_LAYOUT_TILE32) unless --no-tc; everything else on the CUDA-core kernel (COL4)
        self.tc = (not args.no_tc) and self.B >= 4 and ww.tc_workspace_bytes(max(self.nloc, 1), spec.m, self.B) > 0
        layout = ww.LAYOUT_TILE32 if self.tc else ww.LAYOUT_COL4
        nb = ww.packed_bytes(max(self.nloc, 1), spec.m, layout)
        self.R = max(1, int(np.ceil(4 * L2_BYTES / max(nb, 1))))
        planes = torch.empty((4, max(self.nloc, 1), spec.m), dtype=torch.int8, device=dev)
        for q in range(4):
            wi.codes_device(args.seed, q, self.nloc, spec.m, planes[q], spec.dist, row0=sh.row_begin)
        base = ww.pack_ternary_device(planes, layout=layout)
        self.Wr = torch.empty((self.R, nb), dtype=torch.uint8, device=dev)
        self.Wr[:] = base
        sc = wi.scales(args.seed, spec.n, spec.per_row, spec.scale_lo, spec.scale_hi)
        if spec.per_row:
            sc = sc[sh.row_begin:sh.row_end]
        self.S = torch.from_numpy(np.ascontiguousarray(sc)).to(dev)
        self.X = torch.from_numpy(wi.activations(args.seed, spec.m, self.B)).to(dev)
        self.Y = [torch.zeros(sh.n_padded * self.B, dtype=torch.complex64, device=dev)]
        self.L = ww.Layer(self.nloc, spec.m, layout,
                          ww.SCALES_PER_ROW if spec.per_row else ww.SCALES_PER_TENSOR,
                          ww.CONV_EQ1, 0 if args.no_pdl else ww.FLAG_PDL)
        self.ws = (torch.zeros(ww.tc_workspace_bytes(self.nloc, spec.m, self.B) + 256, dtype=torch.uint8, device=dev)
                   if self.tc else None)

    def inputs(self):
        return self.X

    def step(self, s):
        rpr = self.shard.rows_per_rank
        yv = self.Y[0][self.rank * self.B * rpr:(self.rank + 1) * self.B * rpr].view(self.B, rpr)
        for r in range(self.R):
            if self.tc:  # the batch as a dense contraction on the tensor cores
                self.ww.wl_gemv_batched_tc(self.L, self.Wr[r], self.S, self.X, yv, self.ws, stream=s)
            else:
                self.ww.wl_gemv_batched(self.L, self.Wr[r], self.S, self.X, yv, stream=s)
            if self.world > 1:
                import torch.distributed as dist
                n = self.Y[0].numel() // self.world
                dist.all_gather_into_tensor(self.Y[0], self.Y[0][self.rank * n:(self.rank + 1) * n],
                                            group=self.group)
        # the tensor-core path is two launches per layer (x limbs, then the MMA kernel)
        return self.R * (2 if self.tc else self.ww.launches_for_batch(self.B))

    def algorithmic_bytes(self):
        m, n, B = self.spec.m, self.nloc, self.B
        return self.R * (n * self.ww.packed_bytes(1, m) + 8 * m * B + 8 * n * B + 16 * n)

    def packed_act_bytes(self):
        return self.R * (self.nloc * self.ww.packed_bytes(1, self.spec.m) + 8 * self.spec.m * self.B)

    def adds(self):
        return self.R * 8 * self.nloc * self.spec.m * self.B


def launch_plan(gpus: int, env) -> tuple:
    """How to honour --gpus N: ("run", world) in this process (WORLD_SIZE already set by
    torchrun, or N = 1), ("spawn", N) to relaunch under torch.distributed.run with N ranks,
    or ("error", why) when --gpus disagrees with an existing WORLD_SIZE."""
    if gpus < 1:
        return ("error", f"--gpus {gpus} < 1")
    ws = env.get("WORLD_SIZE")
    if ws is None:
        return ("run", 1) if gpus == 1 else ("spawn", gpus)
    if int(ws) != gpus:
        return ("error", f"--gpus {gpus} but WORLD_SIZE={ws} (launch N ranks for --gpus N)")
    return ("run", int(ws))


def spawn_cmd(nproc: int, argv, port: int) -> list:
    """torchrun command line that relaunches this script with nproc ranks on 127.0.0.1."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
            f"--nproc-per-node={nproc}", "--master-addr=127.0.0.1", f"--master-port={port}",
            os.path.abspath(__file__)] + list(argv)


def _free_port() -> int:
    import socket
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def main():
    ap = argparse.ArgumentParser(description=__doc__.split("\n\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--workload", choices=("c4", "c1", "c2", "c3a", "c3b", "c5"), default="c4")
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--no-fuse", action="store_true",
                    help="c4: one launch per projection instead of one per shared input")
    ap.add_argument("--engine", choices=("pdl", "program"), default="pdl",
                    help="c4: PDL-chained launches per stage, or one persistent program launch")
    ap.add_argument("--chain", choices=("plain", "block"), default="plain",
                    help="c4 program: independent seeded stage inputs, or NEXT-3 decode blocks")
    ap.add_argument("--no-x-l2-persist", dest="x_l2_persist", action="store_false",
                    help="do not keep the step's input activations persisting in L2 (default: keep "
                         "them, ww_stream_keep_in_l2, so the H2D-fed inputs of the e2e leg stay "
                         "L2-resident while the weights stream)")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-pdl", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--lut-stages", default="auto",
                    help="c4, pdl engine, plain chain, B = 1: comma-separated stages (qkv,o,gateup,down) "
                         "on the lookup path ww_wl_gemv_lut; 'auto' = all four (a chain mixing the two kernels "
                         "is slower than either, profiles/r02/lut_stage_sets.txt), 'none' = all on the "
                         "predicated-FADD2 kernel")
    ap.add_argument("--no-tc", action="store_true",
                    help="single-layer workloads: keep B >= 4 on the predicated-FADD2 kernel instead "
                         "of the tcgen05 path")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3  # contract: W >= 3
    kind, what = launch_plan(args.gpus, os.environ)
    if kind == "error":
        print(f"bench.py: {what}", file=sys.stderr)
        sys.exit(2)
    if kind == "spawn":
        if args.impl == "ours":
            import torch
            if torch.cuda.device_count() < what:
                print(f"bench.py: --gpus {what} but only {torch.cuda.device_count()} visible "
                      "CUDA devices", file=sys.stderr)
                sys.exit(2)
        sys.exit(subprocess.call(spawn_cmd(what, sys.argv[1:], _free_port())))
    if args.impl == "reference":
        # the oracle runs on rank 0's host cores; other ranks exit 0 without work
        run_reference(args, int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")))
        return
    world, rank, local = _dist_init(args)
    run_ours(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
