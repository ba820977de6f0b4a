#!/usr/bin/env python
"""Benchmark: training graphs/s of the PNA-GCNN step on B200 (BASELINE.json metric).

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference] [--workload B|A|D|E256|E512]

One process per GPU (torchrun for N > 1; RANK / LOCAL_RANK / WORLD_SIZE from the
env). A *step* = one pass of the whole hot path: batch
of B graphs -> 6 GC layers -> pool -> head -> MSE -> backward -> NCCL gradient
mean -> fused AdamW, replayed as one CUDA graph.

Prints ONE JSON line on rank 0:
  value   graphs/s over all ranks, inputs resident in HBM (K pre-packed batches
          in device slots), L2 flushed (512 MB write) between timed steps,
          each step bracketed by CUDA events on the compute stream, max over ranks.
  e2e     the same metric through the public C-ABI from HOST buffers: per step
          hg_pack (host collate from the Table-1 store -> pinned -> H2D),
          hg_train_step, hg_loss_get (D2H of the loss).
  roofline / phases_ms from an instrumented eager step (hg_profile_step).
  cpu_baseline: the float64 oracle (oracle/) timed on a bounded sample (rank 0, N=1).
--impl reference runs the oracle itself as the reference arm (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# NCCL's own log lines (e.g. NCCL_DEBUG=VERSION) go to stderr: stdout carries ONE JSON line
os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")

METRIC = "train graphs/sec at 1/2/4/8 B200 (PCQM4Mv2-shaped); % HBM/tensor roofline"

WORKLOADS = {
    # name: (preset, graphs in store, B per GPU, H, L, description)
    "A": ("tiny", 1000, 64, 32, 2, "A: 1,000 synthetic molecules (<=20 atoms), 2 conv layers hidden 32, batch 64"),
    "B": ("pcqm", 3_400_000, 128, 128, 6,
          "B: PCQM4Mv2-shaped 3.4M synthetic molecules (<=51 atoms), 6 conv layers hidden 128, batch 128/GPU"),
    "D": ("aisd", 10_500_000, 512, 128, 6,
          "D: AISD HOMO-LUMO-shaped 10.5M synthetic molecules, 6 conv layers hidden 128, batch 512/GPU"),
    "E256": ("aisd", 10_500_000, 512, 256, 8, "E: AISD-shaped, 8 conv layers hidden 256, batch 512/GPU"),
    "E512": ("aisd", 10_500_000, 512, 512, 8, "E: AISD-shaped, 8 conv layers hidden 512, batch 512/GPU"),
    # the paper's own model widths (channel-padded internally, include/hgnn.h hg_config_internal)
    "P55": ("pcqm", 3_400_000, 128, 55, 6,
            "paper scalability model (PAPER.md:315): PCQM4Mv2-shaped 3.4M molecules, 6 PNA layers of 55 neurons, "
            "local batch 128"),
    "P200": ("pcqm", 3_400_000, 128, 200, 6,
             "paper convergence-test width (PAPER.md:318): PCQM4Mv2-shaped 3.4M molecules, 6 PNA layers of 200 "
             "neurons, local batch 128"),
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="B", choices=list(WORKLOADS))
    ap.add_argument("--graphs", type=int, default=0, help="override the store size")
    ap.add_argument("--flush-mb", type=int, default=512)
    ap.add_argument("--resident", type=int, default=32, help="distinct pre-packed batches resident in HBM")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--store-dir", default="")
    ap.add_argument("--seed", type=int, default=11)
    ap.add_argument("--precision", default="3xtf32", choices=["3xtf32", "tf32"],
                    help="GEMM precision: 3xTF32 (fp32-accurate, default) or single-pass TF32 (HG_FLAG_TF32)")
    ap.add_argument("--variant", default="base", choices=["base", "self", "scalers5", "nodehead", "all"],
                    help="(f)3 model variants: PNA self-term, all five scalers, node-level head")
    ap.add_argument("--exchange", default="p2p", choices=["p2p", "nccl"],
                    help="N>1 gradient exchange: fused peer-memory reduce/AdamW/all-gather kernel or bucketed NCCL")
    return ap.parse_args()


def mem_available_bytes() -> int:
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemAvailable:"):
                    return int(line.split()[1]) * 1024
    except OSError:
        pass
    return 0


def store_dir(args, preset, n):
    if args.store_dir:
        return args.store_dir
    need = n * (60 * 136 + 120)  # generous bytes/graph estimate
    for base in ("/dev/shm", "/tmp"):
        try:
            st = os.statvfs(base)
            if st.f_bavail * st.f_frsize > need * 1.2:
                return os.path.join(base, f"hgnn_store_{preset}_{n}_{args.seed}")
        except OSError:
            continue
    return os.path.join("/tmp", f"hgnn_store_{preset}_{n}_{args.seed}")


class Clocks:
    """nvidia-smi sampler for the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = f"/tmp/hgnn_clocks_{os.getpid()}.csv"

    def start(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits", "-lms",
                                          "100", "-i", str(self.index)], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self) -> dict:
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        self.proc.wait()
        self.f.close()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as f:
            for line in f:
                p = [t.strip() for t in line.split(",")]
                if len(p) < 9:
                    continue
                try:
                    sm.append(float(p[1]))
                    mx.append(float(p[2]))
                except ValueError:
                    continue
                for nm, v in zip(names, p[5:9]):
                    if v.lower() == "active":
                        reasons.add(nm)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------------ oracle timing
def oracle_rate(data, ids_list, cfg, delta, seconds, max_steps=None):
    """Oracle train steps over the given batches until `seconds` elapse; graphs/s."""
    import oracle as O
    params = O.init_params(cfg, 2)
    st = O.zero_state(params)
    t0 = time.perf_counter()
    graphs = 0
    steps = 0
    for ids in ids_list:
        params, st, _, _ = O.train_step(params, st, data, ids, cfg, delta)
        graphs += len(ids)
        steps += 1
        if time.perf_counter() - t0 > seconds or (max_steps and steps >= max_steps):
            break
    dt = time.perf_counter() - t0
    return graphs / dt, graphs, steps, dt


def cpu_info() -> dict:
    """CPU model (/proc/cpuinfo) and the BLAS numpy runs on (threadpoolctl)."""
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    blas = "unknown"
    try:
        from threadpoolctl import threadpool_info
        b = [i for i in threadpool_info() if i.get("user_api") == "blas"]
        if b:
            blas = f"{b[0].get('internal_api')} {b[0].get('version')} ({b[0].get('num_threads')} threads)"
    except Exception:
        pass
    return {"cpu_model": model, "blas": blas}


def oracle_config_a_epoch() -> dict:
    """the oracle over one full config-A epoch (1,000 molecules <= 20 atoms, L=2,
    H=32, batch 64: 15 steps, drop-last)."""
    import molgen
    import oracle as O
    data = molgen.generate("tiny", 1000, 1)
    delta = O.degree_stat(data)
    cfg = {"f_node": data["f_node"], "f_edge": 4, "hidden": 32, "layers": 2, "fc_hidden": 32}
    params = O.init_params(cfg, 2)
    st = O.zero_state(params)
    ids = O.shard(3, 0, 0, 1, 1000)
    t0 = time.perf_counter()
    for k in range(len(ids) // 64):
        params, st, _, _ = O.train_step(params, st, data, ids[k * 64:(k + 1) * 64], cfg, delta)
    dt = time.perf_counter() - t0
    return {"steps": len(ids) // 64, "seconds": dt, "graphs_per_s": (len(ids) // 64) * 64 / dt}


def blas_threads() -> int:
    try:
        from threadpoolctl import threadpool_info
        info = threadpool_info()
        n = [i.get("num_threads", 1) for i in info if i.get("user_api") == "blas"]
        return max(n) if n else 1
    except Exception:
        return len(os.sched_getaffinity(0))


# ------------------------------------------------------------------------ main
def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    preset, n_graphs, B, H, L, desc = WORKLOADS[args.workload]
    if args.graphs:
        n_graphs = args.graphs
    import numpy as np

    if args.impl == "reference":
        return run_reference(args, rank, world, preset, n_graphs, B, H, L, desc)

    # stdout carries exactly ONE JSON line: anything libraries print while we run
    # (e.g. "NCCL version ...") is routed to stderr until the result is printed
    sys.stdout.flush()
    saved_stdout = os.dup(1)
    os.dup2(2, 1)

    import torch
    import torch.distributed as dist
    import molgen
    from paper_2207_11333_b200 import hgnn

    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local_rank}"))

    def barrier():
        if world > 1:
            dist.barrier()

    # ---- dataset: generated once per host into shared memory-mapped files
    mem_need = n_graphs * 5600 * (2.0 if preset == "aisd" else 1.0)
    avail = mem_available_bytes()
    if avail and mem_need > 0.6 * avail:
        scaled = int(n_graphs * 0.6 * avail / mem_need)
        log(f"[bench] host memory {avail / 1e9:.1f} GB: store reduced {n_graphs} -> {scaled} graphs")
        n_graphs = scaled
    sdir = store_dir(args, preset, n_graphs)
    t0 = time.time()
    if local_rank == 0:
        data = molgen.generate_to(sdir, preset, n_graphs, args.seed)
    barrier()
    if local_rank != 0:
        data = molgen.load_dir(sdir)
    t_gen = time.time() - t0
    t0 = time.time()
    if args.variant in ("nodehead", "all"):  # node-level targets: seeded synthetic, one per atom
        data = dict(data)
        data["y_node"] = np.random.default_rng(args.seed).standard_normal(len(data["x"])).astype(np.float32)
    store = hgnn.Store(data, copy=False)
    st = store.stats()
    delta = store.degree_stat()
    t_store = time.time() - t0
    log(f"[bench] rank {rank}: store {st} delta={delta:.6f} gen {t_gen:.1f}s store {t_store:.1f}s")

    max_nodes = B * st["max_nodes_per_graph"]
    max_edges = B * int(np.diff(np.asarray(data["edge_offset"])).max())
    n_res = max(1, min(args.resident, args.steps))
    e2e_slots = 0 if args.no_e2e else 2
    flags = hgnn.HG_FLAG_TF32 if args.precision == "tf32" else 0
    scalers = 0
    if args.variant in ("self", "all"):
        flags |= hgnn.HG_FLAG_SELF_TERM
    if args.variant in ("nodehead", "all"):
        flags |= hgnn.HG_FLAG_NODE_HEAD
    if args.variant in ("scalers5", "all"):
        scalers = sum(hgnn.SCALER_BITS.values())
    cfg = hgnn.make_config(data["f_node"], 4, H, L, B, max_nodes, max_edges, delta, n_slots=n_res + e2e_slots,
                           max_degree=st["max_degree"], flags=flags, scalers=scalers,
                           delta_lin=store.degree_stat_linear() if scalers else 0.0)
    ctx = hgnn.Context(cfg, device=local_rank)
    ctx.params_init(1234)
    ctx.comm_init(rank, world)
    exchange = args.exchange if world > 1 else "none"
    if exchange == "p2p":
        try:
            ctx.p2p_init(rank, world)
        except hgnn.HgError as e:  # e.g. a workspace that is not cudaMalloc-backed: NCCL buckets
            log(f"rank {rank}: peer-memory exchange unavailable ({e}); using the NCCL exchange")
            exchange = f"nccl (p2p unavailable: {e})"
        # (p2p_init agrees across ranks: all take the peer-memory path or none)
    hyper = dict(hgnn.DEFAULT_ADAMW)
    # host collation threads: 4 on one GPU; with W ranks sharing the host, cores / W each
    pack_threads = max(1, len(os.sched_getaffinity(0)) // world) if world > 1 else 4
    hgnn.pack_threads_set(pack_threads)

    ids = hgnn.hg_shard(13, 0, rank, world, n_graphs)
    nb = len(ids) // B
    batches = [ids[k * B:(k + 1) * B] for k in range(nb)]
    blobs = [hgnn.hg_pack_host(store, batches[k % nb], cfg) for k in range(n_res)]
    for s, blob in enumerate(blobs):
        ctx.upload(blob, s)
    for s in range(n_res + e2e_slots):
        ctx.capture_step(s, **hyper)
    stream = torch.cuda.current_stream()
    flush = torch.empty(args.flush_mb << 20, dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()

    # ---- warm-up
    for k in range(args.warmup):
        ctx.train_step(k % n_res, graph=True, **hyper)
    torch.cuda.synchronize()
    barrier()

    # ---- timed: device-resident inputs
    K = args.steps
    ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    clocks = Clocks(local_rank)
    clocks.start()
    l0 = ctx.launch_count()
    barrier()
    torch.cuda.synchronize()
    for k in range(K):
        flush.zero_()
        ev0[k].record(stream)
        ctx.train_step(k % n_res, graph=True, **hyper)
        ev1[k].record(stream)
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    launches = ctx.launch_count() - l0
    total_ms = sum(a.elapsed_time(b) for a, b in zip(ev0, ev1))
    tmax = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    total_ms = float(tmax.item())
    value = world * K * B / (total_ms / 1e3)
    loss_now = ctx.loss()

    # ---- forward-only evaluation over the resident batches: device-timed
    ctx.eval_reset()
    for s in range(n_res):  # capture the eval graphs, warm
        ctx.eval_batch(s)
    ctx.eval_reset()
    barrier()
    torch.cuda.synchronize()
    ev_a, ev_b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev_a.record(stream)
    for k in range(K):
        ctx.eval_batch(k % n_res)
    ev_b.record(stream)
    torch.cuda.synchronize()
    em = ev_a.elapsed_time(ev_b)
    tm = torch.tensor([em], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
    em = float(tm.item())
    er = ctx.eval_result()
    eval_out = {"value": world * K * B / (em / 1e3), "unit": "graphs/s", "ms_per_batch": em / K,
                "mse": er["mse"], "mae": er["mae"], "graphs": er["count"],
                "note": "hg_eval_batch (forward + fp64 MSE/MAE accumulation, graph replay) over the resident "
                        "batches, device-timed, no L2 flush; metrics of the trained-for-a-few-steps model"}

    # ---- e2e through the public API from host buffers
    e2e = None
    if not args.no_e2e:
        s0 = n_res
        off = n_res * 0
        for k in range(2):  # warm the e2e slots
            ctx.pack(store, batches[(off + k) % nb], s0 + (k % 2))
            ctx.train_step(s0 + (k % 2), graph=True, **hyper)
            ctx.loss()
        h2d = []
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ctx.pack(store, batches[(n_res + 2) % nb], s0)
        h2d.append(int(hgnn.hg_batch_offsets(B, 0, 0, 0, 0)["total"]))
        losses = []
        for k in range(K):
            slot = s0 + (k % 2)
            ctx.train_step(slot, graph=True, **hyper)
            ctx.loss_enqueue(k % 4)  # D2H read of this step's loss into pinned memory (async)
            if k + 1 < K:
                nxt = batches[(n_res + 3 + k) % nb]
                ctx.pack(store, nxt, s0 + ((k + 1) % 2))
            if k > 0:
                losses.append(ctx.loss_fetch((k - 1) % 4))  # previous step's loss, already copied
        losses.append(ctx.loss_fetch((K - 1) % 4))
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        barrier()
        tt = torch.tensor([dt], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dt = float(tt.item())
        # exact H2D bytes per step: the packed blob sizes
        sizes = [hgnn.hg_pack_host(store, batches[(n_res + 2 + k) % nb], cfg).nbytes for k in range(min(K, 8))]
        e2e = {"value": world * K * B / dt, "unit": "graphs/s", "h2d_bytes_per_step": int(np.mean(sizes)),
               "d2h_bytes_per_step": 4, "ms_per_step": dt * 1e3 / K,
               "note": "hg_pack (host collate + pinned H2D, overlapped with the previous step) + hg_train_step "
                       "(graph) + hg_loss_enqueue/hg_loss_fetch (every step's loss read back to the host, "
                       "consumed one step later); wall clock, max over ranks"}

    # ---- instrumented step: per-phase device time -> roofline of the dominant kernel
    prof = None
    phases = {}
    reps = 3
    for r in range(reps):
        flush.zero_()
        p = ctx.profile_step(r % n_res, **hyper)
        for k, (ms, nl) in p.items():
            a = phases.setdefault(k, [0.0, 0])
            a[0] += ms / reps
            a[1] = nl
    # algorithmic work per phase:
    # bytes = compulsory fp32 traffic of the method per node-layer, flops = fp32 MACs x 2
    Ns, Es = [], []
    for r in range(reps):
        hdr = blobs[r % n_res][:64].view(np.int32)
        Ns.append(int(hdr[1]))
        Es.append(int(hdr[2]))
    Nn, Ee = float(np.mean(Ns)), float(np.mean(Es))
    eb = Ee / Nn  # mean in-degree
    F0 = data["f_node"]
    NL, NL1 = Nn * L, Nn * (L - 1)  # node-layers, node-layers with F = H
    work = {  # phase -> (algorithmic bytes, algorithmic flops)
        "proj": (Nn * (4 * F0 + 4 * H) + NL1 * 8 * H, 2.0 * Nn * H * F0 + 2.0 * NL1 * H * H),
        "agg_fwd": (NL * (22 * H + 4 + 20 * eb), 0.0),
        "update": (NL * (20 * H + 8), 8.0 * NL * H * H),
        "dA": (NL * 20 * H, 8.0 * NL * H * H),
        "dU": (NL * 20 * H, 8.0 * NL * H * H + NL * H),
        "agg_bwd": (NL * (34 * H + 4 + 20 * eb), 0.0),
        "dMx": (Nn * (4 * H + 4 * F0) + NL1 * 8 * H, 2.0 * Nn * H * (F0 + 1) + 2.0 * NL1 * H * (H + 1)),
        "dX": (NL1 * 12 * H, 2.0 * NL1 * H * H),
    }
    # SURVEY §8(d)'s counting of the same phases: the update and its backward as the 12H-wide
    # scaler concatenation would compute them (24H^2 FLOPs per node-layer each for update, dA, dU);
    # the kernels execute the exact degree-class reassociation (8H^2 each), so "executed" is
    # the work the tensor pipe does and "s8" the method's nominal work
    work_s8 = dict(work)
    work_s8["update"] = (work["update"][0], 24.0 * NL * H * H)
    work_s8["dA"] = (work["dA"][0], 24.0 * NL * H * H)
    work_s8["dU"] = (work["dU"][0], 24.0 * NL * H * H + NL * H)
    # fused dX -> dA kernel (k_dxda): the dA of layers < L-1 runs inside the dX phase
    n_da = phases.get("dA", [0.0, L])[1]
    if "dA" in phases and 0 < n_da < L:
        for w in (work, work_s8):
            (ba, fa), (bx, fx) = w["dA"], w["dX"]
            w["dA"] = (ba * n_da / L, fa * n_da / L)
            w["dX"] = (bx + ba * (L - n_da) / L, fx + fa * (L - n_da) / L)
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except OSError:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    bf16_peak = float(peaks.get("bf16_tflops", 2250.0))
    # 3xTF32: three tf32 MMAs per fp32 MAC; tf32 dense = bf16 dense x 0.5 (nominal ratio, B200_PROFILING.md)
    passes = 1 if args.precision == "tf32" else 3
    tc_peak = bf16_peak * 0.5 / passes
    tc_peak_source = ("MEASURED_PEAKS.json bf16_tflops x 0.5 (tf32, single pass)" if passes == 1 else
                      "MEASURED_PEAKS.json bf16_tflops x 0.5 (tf32) / 3 (3xTF32 passes)")
    ridge = tc_peak * 1e12 / (hbm_peak * 1e9)  # flop / byte
    step_ms_prof = sum(v[0] for v in phases.values())
    traffic_db = {}  # this workload's ncu DRAM read + write bytes per launch (tools/traffic_from_ncu.py)
    try:
        with open(os.path.join(ROOT, "profiles", "traffic_per_launch.json")) as f:
            traffic_db = json.load(f).get(args.workload, {})
        if not isinstance(traffic_db, dict) or args.precision != "3xtf32" or args.variant != "base":
            traffic_db = {}  # (captured for the base model in 3xTF32 only)
    except (OSError, ValueError, AttributeError):
        pass

    def roof(k):
        byt, fl = work[k]
        t = phases[k][0] / 1e3
        launches_k = max(1, phases[k][1])
        if fl > 0 and fl / byt >= ridge:
            ach = fl / t / 1e12
            r = {"bound": "tensor", "achieved": ach, "peak": tc_peak, "unit": "TFLOP/s", "frac": ach / tc_peak,
                 "peak_source": tc_peak_source}
        else:
            ach = byt / t / 1e9
            r = {"bound": "hbm", "achieved": ach, "peak": hbm_peak, "unit": "GB/s", "frac": ach / hbm_peak,
                 "peak_source": "MEASURED_PEAKS.json hbm_gbs"}
        r.update({"kernel": k, "ms": phases[k][0], "launches": phases[k][1],
                  "algorithmic_bytes_per_launch": byt / launches_k, "algorithmic_flops_per_launch": fl / launches_k,
                  "intensity_flop_per_byte": fl / byt, "share_of_step": phases[k][0] / step_ms_prof,
                  "traffic": traffic_db.get(k)})
        if r["bound"] == "tensor":
            fl8 = work_s8[k][1]
            r.update({"flops_counting": "executed: degree-class form (8H^2 per node-layer per update/dA/dU GEMM)",
                      "achieved_s8": fl8 / t / 1e12, "frac_s8": fl8 / t / 1e12 / tc_peak,
                      "flops_counting_s8": "SURVEY §8(d): 24H^2 per node-layer per update/dA/dU GEMM",
                      "algorithmic_flops_per_launch_s8": fl8 / launches_k})
        return r

    dom = max((k for k in phases if k in work), key=lambda k: phases[k][0])
    prof = roof(dom)
    phase_roof = {k: {kk: (round(vv, 4) if isinstance(vv, float) else vv) for kk, vv in roof(k).items()
                      if kk in ("bound", "achieved", "frac", "frac_s8", "ms", "intensity_flop_per_byte")}
                  for k in work if k in phases}
    # the north_star's aggregation bar (>= 60% of HBM): algorithmic bytes / time
    agg = {k: {"algorithmic_GBps": round(work[k][0] / (phases[k][0] / 1e3) / 1e9, 1),
               "frac_of_hbm": round(work[k][0] / (phases[k][0] / 1e3) / 1e9 / hbm_peak, 4),
               "us_per_launch": round(1e3 * phases[k][0] / max(1, phases[k][1]), 2),
               "bytes_per_node_layer": f"{'22' if k == 'agg_fwd' else '34'}H + 4 + 20*ebar"}
           for k in ("agg_fwd", "agg_bwd") if k in phases}

    # ---- host-only collation rate (SURVEY §8(d) timing protocol (3)): hg_pack_host from the store
    nb_pack = min(nb, 200)
    t0 = time.perf_counter()
    for k in range(nb_pack):
        hgnn.hg_pack_host(store, batches[k], cfg)
    dtp = time.perf_counter() - t0
    pack_rate = {"graphs_per_s_per_rank": nb_pack * B / dtp, "threads": pack_threads, "batches": nb_pack,
                 "note": "hg_pack_host (C++ collate of B graphs from the Table-1 store), host only"}

    # ---- exchange alone (N > 1): peer-memory exchange or NCCL bucketed path, bus GB/s
    exch = None
    if world > 1:
        import torch.distributed as tdist
        P4 = ctx.n_params * 4
        busf = 2.0 * (world - 1) / world
        exch = {"grad_bytes": P4, "bus_factor": busf, "nvlink_ref_GBps": 770.0,
                "nvlink_ref_source": "B200_PROFILING.md peer copy per direction (900 nominal)"}
        barrier()
        t_ex = ctx.exchange_time(20, **hyper)
        barrier()
        exch["step_exchange"] = {"kind": exchange, "ms": t_ex, "busbw_GBps": P4 * busf / (t_ex / 1e3) / 1e9}
        sweep = {}
        for sz in [64 << 10, 256 << 10, 1 << 20, 4 << 20, 16 << 20, 64 << 20, 128 << 20]:
            tsw = torch.empty(sz // 4, dtype=torch.float32, device="cuda")
            for _ in range(3):
                tdist.all_reduce(tsw)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                tdist.all_reduce(tsw)
            e1.record()
            torch.cuda.synchronize()
            tt = e0.elapsed_time(e1) / 10
            sweep[str(sz)] = {"ms": tt, "busbw_GBps": sz * busf / (tt / 1e3) / 1e9}
            del tsw
        exch["nccl_allreduce_sweep"] = sweep
        bucket_sizes = [4 * (e - b0) for b0, e in hgnn.bucket_layout(cfg)]
        exch["nccl_bucket_bytes"] = bucket_sizes

    # ---- CPU baseline: the oracle on a bounded sample (rank 0, N = 1)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        ocfg = {"f_node": data["f_node"], "f_edge": 4, "hidden": H, "layers": L, "fc_hidden": H}
        sample_batches = [np.asarray(batches[k]) for k in range(min(nb, 64))]
        sub = {k: np.asarray(data[k]) if k in ("node_offset", "edge_offset", "y") else data[k]
               for k in ("node_offset", "edge_offset", "x", "edge_index", "edge_attr", "y")}
        rate, g, s, dt = oracle_rate(sub, sample_batches, ocfg, delta, args.cpu_seconds)
        cpu = {"value": rate, "unit": "graphs/s", "cores": blas_threads(), "kind": "oracle",
               "sample": f"{s} oracle train steps (f64 numpy forward+backward+AdamW) on batches of {B} graphs of "
                         f"this workload, {dt:.1f} s", "host_cores": len(os.sched_getaffinity(0))}
        cpu.update(cpu_info())
        cpu["config_A_epoch"] = oracle_config_a_epoch()

    out = {
        "metric": METRIC, "value": value, "unit": "graphs/s", "n_gpus": world, "steps": K, "warmup": args.warmup,
        "ms_per_step": total_ms / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "tf32" if args.precision == "tf32" else "f32", "data": "synthetic (molgen seeded molecules, Table-2 calibrated; random-init weights)",
        "config": {"workload": desc, "graphs_in_store": n_graphs, "global_batch": B * world, "batch_per_gpu": B,
                   "layers": L, "hidden": H, "hidden_internal": int(ctx.internal_cfg.hidden),
                   "nodes_per_batch_mean": Nn, "edges_per_batch_mean": Ee,
                   "parallelism": f"dp{world}", "resident_batches": n_res,
                   "grad_exchange": exchange,
                   "l2": f"flushed between timed steps ({args.flush_mb} MB write, outside the step events)",
                   "gemm_precision": ("single-pass TF32 tcgen05 (HG_FLAG_TF32), degree-class GEMMs, TMA-fed"
                                      if args.precision == "tf32" else
                                      "3xTF32 tcgen05 (fp32-accurate), degree-class GEMMs, TMA-fed"),
                   "variant": {"name": args.variant, "flags": flags, "scalers": list(hgnn.scaler_names(scalers))
                               if scalers else ["identity", "amplification", "attenuation"],
                               "work_accounting": "base model terms (variant extra terms not counted)"
                               if args.variant != "base" else "base model"}},
        "roofline": prof, "phase_roofline": phase_roof, "aggregation": agg, "pack_rate": pack_rate,
        "exchange": exch,
        "phases_ms": {k: round(v[0], 4) for k, v in phases.items()},
        "phase_launches": {k: v[1] for k, v in phases.items()},
        "cpu_baseline": cpu, "e2e": e2e, "eval": eval_out, "gpu_launches": launches, "clocks": clk,
        "loss_after_timed": loss_now,
    }
    sys.stdout.flush()
    os.dup2(saved_stdout, 1)
    if rank == 0:
        print(json.dumps(out), flush=True)
    os.dup2(2, 1)
    barrier()
    if world > 1:
        dist.destroy_process_group()


def run_reference(args, rank, world, preset, n_graphs, B, H, L, desc):
    """Reference arm = the float64 CPU oracle as it stands (rank 0 only), on this arm's workload:
    the same seeded store, the same rank-0 shard, full B-graph batches; each step is one oracle
    train step (forward, backward, AdamW) of one batch."""
    import numpy as np
    if rank != 0:
        return
    import molgen
    import oracle as O
    t0 = time.time()
    data = molgen.generate_to(store_dir(args, preset, n_graphs), preset, n_graphs, args.seed)
    ids = O.shard(13, 0, 0, world, n_graphs)
    # delta over a bounded sample of the training graphs (the oracle's per-graph loop over the
    # whole store would take minutes; the value only scales the scalers)
    delta = O.degree_stat(data, ids[:20000])
    log(f"[bench] reference: store {n_graphs} graphs in {time.time() - t0:.1f}s, delta={delta:.6f}")
    ocfg = {"f_node": data["f_node"], "f_edge": 4, "hidden": H, "layers": L, "fc_hidden": H}
    batches = [ids[k * B:(k + 1) * B] for k in range(args.warmup + args.steps)]
    params = O.init_params(ocfg, 2)
    st = O.zero_state(params)
    for k in range(args.warmup):
        params, st, _, _ = O.train_step(params, st, data, batches[k], ocfg, delta)
    t0 = time.perf_counter()
    for k in range(args.steps):
        params, st, _, _ = O.train_step(params, st, data, batches[args.warmup + k], ocfg, delta)
    dt = time.perf_counter() - t0
    value = args.steps * B / dt
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": "graphs/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3 / args.steps,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (molgen seeded molecules, Table-2 calibrated; random-init weights)",
           "config": {"workload": desc, "graphs_in_store": n_graphs, "global_batch": B * world, "batch_per_gpu": B,
                      "layers": L, "hidden": H, "parallelism": "cpu oracle (f64 numpy), rank 0 only"},
           "cpu_baseline": {"value": value, "unit": "graphs/s", "kind": "oracle", "cores": blas_threads(),
                            "sample": f"{args.steps} oracle train steps of {B}-graph batches (rank 0's shard of "
                                      f"the {n_graphs}-graph store; delta over 20000 of its graphs)"},
           "e2e": {"value": value, "unit": "graphs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
