"""bench.py — batched XOR-PIR server scan on B200 (BASELINE.json config 4).

Workload (one "step"): a batch of 8,192 PIR requests, each a 2^20-bit bucket-
selection vector expanded on device from a 16-byte seed (zero-extended to the
reference's 32-byte PRG seed, crypto.hpp:20) with the reference's ChaCha20 PRG,
answered against a 4 GiB store (1,048,576 buckets x 4 x 1,024-byte slots) of
DetRng(3) bytes, bucket-range sharded over the N ranks, partial answers
XOR-reduced over NVLink peer memory (fused into the scan epilogue: each rank's
accumulator flushes are peer atomics into the row owner's buffer). Everything is generated on device from the
recipe in SURVEY.md §8(d); data = synthetic.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line on rank 0 (bench contract in the task statement):
  value        whole-job requests/s with seeds + store resident in HBM
  e2e          the same metric through the C-ABI host call xpir_answer_batch_seeded
               (host seeds in, host answers out, copies inside the timed region)
  roofline     dominant kernel (k_scan_m4rm_q9 at config 4) vs the dense-LOP3 ALU bound
  cpu_baseline the reference's pir::answer_batch (oracle/_ref) on the host cores
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

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_BUCKETS = 1 << 20
BUCKET_BYTES = 4096  # depth 4 x 1,024-byte slots
BATCH = 8192
STORE_SEED = 3  # DetRng(3), SURVEY.md §8(d) config 4
METRIC = "PIR requests/sec (batched XOR-PIR scan, 4 GiB store, 8192 seeded requests)"
UNIT = "requests/s"
SAMPLED = os.path.join(ROOT, "tests", "golden", "sampled.json")


def workload_config(batch: int) -> dict:
    """The `config` object both arms print (identical, so the driver can match them)."""
    return {"workload": "config4: 4 GiB store (1,048,576 buckets x 4 x 1,024 B), 8192 seeded requests, "
                        "bucket-range sharded",
            "store_bytes": N_BUCKETS * BUCKET_BYTES, "batch": batch, "buckets": N_BUCKETS,
            "bucket_bytes": BUCKET_BYTES, "l2": "inputs larger than L2 (4 GiB store streamed every step)"}


def sampled_golden():
    """>= 64 reference rows of the bench's exact batch (oracle/make_golden_sampled.py
    over the unmodified reference's pir::answer_batch), or None when the run is
    not the config-4 workload."""
    if N_BUCKETS != 1 << 20 or not os.path.exists(SAMPLED):
        return None
    with open(SAMPLED) as f:
        g = json.load(f)["config4"]
    return g if g["B"] == BATCH else None


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device, self.rows, self.proc = device, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-i", str(self.device),
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if r[3 + k] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ---------------------------------------------------------------------------
# CPU baseline: the reference's pir::answer_batch on host cores (oracle/_ref)
# ---------------------------------------------------------------------------
class CpuReference:
    """The unmodified reference pir::answer_batch (oracle/_ref; the C restatement
    when the reference build is absent) on the host cores: one thread per core,
    each on a disjoint slice of the requests over ONE shared immutable Snapshot
    (concurrent answers are allowed by the reference contract)."""

    def __init__(self):
        import oracle

        self.o = oracle.best()
        self.kind = self.o.kind
        self.threads = os.cpu_count() or 1
        g = self.o.detrng(STORE_SEED)  # call 0 = the 4 GiB store
        if self.kind == "reference":
            self.snap = self.o.snapshot_detrng(g, N_BUCKETS, BUCKET_BYTES)
        else:
            self.db = np.frombuffer(g.fill(N_BUCKETS * BUCKET_BYTES), np.uint8)
        self.q = {}

    def queries(self, B):
        from oracle import recipes

        if B not in self.q:
            seeds = recipes.config4_seeds(self.o, B)
            self.q[B] = np.stack([np.frombuffer(self.o.prng_expand(s.tobytes(), N_BUCKETS // 8), np.uint8)
                                  for s in seeds])
        return self.q[B]

    def time(self, B, threads: int | None = None) -> float:
        q = self.queries(B)
        th = self.threads if threads is None else threads
        if self.kind == "reference":
            return self.snap.answer_batch(q, B, th)[1]
        t0 = time.perf_counter()
        self.o.answer_batch(self.db, N_BUCKETS, BUCKET_BYTES, q, B, threads=th)
        return time.perf_counter() - t0

    def calibrate(self, target_s: float, max_per_thread: int = 256) -> int:
        """Requests per sample so one sample takes about target_s."""
        per = 1
        while True:
            secs = self.time(self.threads * per)
            if secs >= target_s / 2 or per >= max_per_thread:
                return self.threads * per
            per = min(max_per_thread, max(per * 2, int(per * target_s / max(secs, 1e-3))))

    def describe(self, B, secs) -> str:
        return (f"{B} of the 8192 config-4 requests (seeds = DetRng(3) calls 1..{B}) over the full 4 GiB "
                f"store, {self.threads} threads x answer_batch slices, {secs:.1f} s per sample")


def cpu_reference_sample(target_s: float = 15.0):
    """All-core rate on a calibrated sample, plus the single-thread rate (the
    reference's answer_batch as it ships, one core) on 4 requests."""
    ref = CpuReference()
    B = ref.calibrate(target_s)
    secs = ref.time(B)
    one = 4 / ref.time(4, threads=1)
    return B / secs, ref.threads, ref.describe(B, secs), ref.kind, one


def run_reference(args):
    rank = env_int("RANK", 0)
    if rank != 0:
        return 0
    ref = CpuReference()
    B = ref.calibrate(args.ref_step_seconds)
    times = []
    for i in range(args.warmup + args.steps):
        secs = ref.time(B)
        if i >= args.warmup:
            times.append(secs)
    secs = statistics.median(times)
    value = B / secs
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * BATCH / value,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic (DetRng / ChaCha20 recipe of SURVEY.md §8(d))",
        "config": workload_config(BATCH),
        "parallelism": f"host threads={ref.threads}",
        "step": f"a bounded sample of {B} requests per step; ms_per_step scaled to the 8192 batch",
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": ref.threads, "kind": ref.kind,
                         "sample": ref.describe(B, secs)},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def traffic_from_profile(n_buckets, batch, world, kernel):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant
    kernel from the committed ncu capture of this same workload (profiles/),
    or None when the capture does not match the configuration being run."""
    name = {5: "r01_traffic_m4rm_tmem", 8: "r02_traffic_m4rm_q9"}.get(kernel)
    path = os.path.join(ROOT, "profiles", f"{name}.json")
    if name is None or world != 1 or n_buckets != 1 << 20 or batch != BATCH or not os.path.exists(path):
        return None
    with open(path) as f:
        t = json.load(f)
    return t["dram_bytes_read"] + t["dram_bytes_write"]


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def main():
    global N_BUCKETS
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=BATCH)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-step-seconds", type=float, default=8.0)
    ap.add_argument("--kernel", type=int, default=0, help="0 auto, 1 direct, 2 m4rm")
    ap.add_argument("--buckets", type=int, default=N_BUCKETS,
                    help="store buckets (profiling runs only; the bench line uses config 4)")
    ap.add_argument("--quick", action="store_true", help="timed steps only (for ncu)")
    args = ap.parse_args()
    N_BUCKETS = args.buckets
    if args.impl == "reference":
        return run_reference(args)

    import torch

    import paper_2001_08250_b200 as xp

    rank, world, local = env_int("RANK", 0), env_int("WORLD_SIZE", 1), env_int("LOCAL_RANK", 0)
    ndev = torch.cuda.device_count()
    # More ranks than GPUs (a 1-GPU development box): ranks share the GPUs and the
    # control plane runs on gloo. Only for validating the multi-rank path — the
    # timings are not scaling numbers and the line says so.
    shared_gpu = world > ndev
    local = local % ndev
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        if shared_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))

    def max_over_ranks(x: float) -> float:
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if shared_gpu else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())
    def sum_over_ranks(x: float) -> float:
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if shared_gpu else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())
    B = args.batch
    xp.set_scan_opts(args.kernel)
    key = xp.blake2b(STORE_SEED.to_bytes(8, "little"), 32)  # DetRng(3) key (rng.cpp:18-23)

    from paper_2001_08250_b200.sharded import ShardedScan, ShardPlan

    plan = ShardPlan(N_BUCKETS, world)
    stream = torch.cuda.Stream()  # a real stream handle (not the legacy default stream)
    torch.cuda.set_stream(stream)
    if world > 1:
        sh = ShardedScan(xp, torch, dist, N_BUCKETS, BUCKET_BYTES, B, local)
        store = sh.store
    else:
        sh = None
        store = xp.Store(N_BUCKETS, BUCKET_BYTES, 0, N_BUCKETS, device=local)
    lo, hi = plan.bucket_range(rank)
    store.fill_keystream(key, 0)  # call 0 of DetRng(3): the shard's window of the 4 GiB store
    seeds = torch.zeros((B, 32), dtype=torch.uint8, device="cuda")
    xp.keystream_rows_dev(key, 1, B, 16, seeds, 32, device=local)  # calls 1..B, 16 B each
    out = torch.empty((B, BUCKET_BYTES), dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()

    own = {"rows": out, "r0": 0}

    def step():
        if sh is not None:
            own["rows"], own["r0"] = sh.step(seeds, stream=stream), sh.r0
        else:
            store.answer_batch_seeded_dev(seeds, B, out, stream=stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    xp.scan_timing_collect()
    xp.scan_timing(True)
    if sh is not None and sh.fused:
        sh.store.peer_stats(reset=True)
    l0 = xp.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
    launches = xp.launch_count() - l0
    xp.scan_timing(False)
    scan_ms, scan_launches = xp.scan_timing_collect()
    ms = max_over_ranks(e0.elapsed_time(e1))
    ms_per_step = ms / args.steps
    value = B / (ms_per_step * 1e-3)

    # bytes the fused epilogue pushed over NVLink per rank per step, against a reduce-scatter's
    peer_bytes = None
    if sh is not None and sh.fused:
        ps = sh.store.peer_stats()
        remote = max_over_ranks(float(ps["remote_bytes"])) / args.steps
        peer_bytes = {"remote_per_rank_per_step_max": remote,
                      "reduce_scatter_bytes_per_rank": B * BUCKET_BYTES * (world - 1) / world,
                      "ratio": remote / (B * BUCKET_BYTES * (world - 1) / world)}

    # parity of the last timed step's output: every reference-sampled row this rank owns
    parity = "unchecked (not the config-4 workload)"
    gold = sampled_golden() if B == BATCH else None
    if gold is not None:
        import hashlib

        torch.cuda.synchronize()
        rows, r0 = own["rows"], own["r0"]
        mine = [(i, r) for i, r in enumerate(gold["rows"]) if r0 <= r < r0 + rows.shape[0]]
        bad = sum(hashlib.sha256(rows[r - r0].cpu().numpy().tobytes()).hexdigest() != gold["out_rows_sha256"][i]
                  for i, r in mine)
        bad, checked = int(sum_over_ranks(float(bad))), int(sum_over_ranks(float(len(mine))))
        parity = ("ok" if bad == 0 else "MISMATCH") + \
            f" ({checked} reference rows of the timed batch, tests/golden/sampled.json; {bad} differ)"

    if args.quick:
        if rank == 0:
            print(json.dumps({"quick": True, "ms_per_step": ms_per_step, "value": value,
                              "scan_ms_per_launch": scan_ms / max(scan_launches, 1),
                              "kernel": xp.last_scan_kernel(), "buckets": N_BUCKETS}), flush=True)
        return 0
    # e2e through the C-ABI host call (host seeds -> device -> host answers)
    e2e = None
    if world == 1:
        # pinned host buffers (the seeds arrive from the network into host memory,
        # the answers leave from it)
        hseeds_t = seeds.cpu().pin_memory()
        hout_t = torch.empty((B, BUCKET_BYTES), dtype=torch.uint8).pin_memory()
        hseeds, hout = hseeds_t.numpy(), hout_t.numpy()
        store.answer_batch_seeded(hseeds, out=hout)  # warm
        t_e2e = []
        for _ in range(max(2, min(args.steps, 3))):
            t0 = time.perf_counter()
            store.answer_batch_seeded(hseeds, out=hout)
            t_e2e.append(time.perf_counter() - t0)
        e2e = {"value": B / statistics.median(t_e2e), "unit": UNIT, "h2d_bytes_per_step": B * 32,
               "d2h_bytes_per_step": B * BUCKET_BYTES,
               "path": "xpir_answer_batch_seeded (pinned host buffers, wall clock)"}
        assert hout.shape == (B, BUCKET_BYTES)
    else:
        # sharded e2e: host seeds H2D on every rank, each rank's owned rows D2H
        hseeds = seeds.cpu().pin_memory()
        r0, r1 = plan.row_range(rank, B)
        hrows = torch.empty((r1 - r0, BUCKET_BYTES), dtype=torch.uint8).pin_memory()
        dseeds = torch.empty_like(seeds)
        t_e2e = []
        for _ in range(max(2, min(args.steps, 3))):
            torch.cuda.synchronize()
            dist.barrier()
            f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            f0.record(stream)
            dseeds.copy_(hseeds, non_blocking=True)
            own = sh.step(dseeds, stream=stream)
            hrows.copy_(own, non_blocking=True)
            f1.record(stream)
            torch.cuda.synchronize()
            t_e2e.append(max_over_ranks(f0.elapsed_time(f1)) * 1e-3)
        e2e = {"value": B / statistics.median(t_e2e), "unit": UNIT, "h2d_bytes_per_step": B * 32,
               "d2h_bytes_per_step": (r1 - r0) * BUCKET_BYTES * world,
               "path": "per-rank seeds H2D + owned answer rows D2H"}

    # roofline of the dominant kernel (k_scan_m4rm_q9 at config 4) on this rank's shard
    peaks = xp.measure_peaks(local)
    nb = hi - lo
    per_launch_ms = scan_ms / max(scan_launches, 1)
    work_lop3 = B * nb * BUCKET_BYTES / 4  # dense select-XOR: one 32-bit LOP3 per (request, bucket, word)
    achieved = work_lop3 / (per_launch_ms * 1e-3)
    hbm_bytes = nb * BUCKET_BYTES + B * (nb // 8) + B * BUCKET_BYTES
    hbm_peak = 6545.0
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            hbm_peak = float(json.load(f)["hbm_gbs"])
            peak_src = "MEASURED_PEAKS.json"
    except Exception:
        peak_src = "fallback 6545 GB/s"
    kernel = xp.last_scan_kernel()
    # shared-memory lookup bytes of the table kernel that ran: 32 B per (request,
    # table, 32-byte column); kernel 8's tables cover 9 buckets (2 sets of 4 tables
    # per 72 buckets), the byte tables 8
    n_tables = 8 * ((nb + 71) // 72) if kernel == 8 else nb // 8
    lookup_bytes = B * n_tables * BUCKET_BYTES
    roof = {
        "bound": "alu",
        "kernel": {1: "k_scan_direct", 2: "k_scan_m4rm", 5: "k_scan_m4rm_tmem",
                   7: "k_scan_m4rm4", 8: "k_scan_m4rm_q9", 9: "k_scan_m4rm6"}.get(kernel, "?"),
        "unit": "Tops/s (32-bit masked-XOR lane ops)",
        "achieved": achieved / 1e12,
        "peak": peaks["lop3_per_s"] / 1e12,
        "frac": achieved / peaks["lop3_per_s"],
        "peak_source": "measured live: k_lop3_peak (acc ^= w & m, 148 SMs)",
        "traffic": traffic_from_profile(N_BUCKETS, B, world, kernel),
        "algorithmic_ops_per_launch": work_lop3,
        "launch_ms": per_launch_ms,
        "note": ("W = B*N_g*S/4 dense GF(2) select-XOR ops; the M4RM kernel does one 32-byte table "
                 "lookup per (request, 9 buckets, 32-byte column) instead (8 buckets for the byte-table "
                 "kernels), so frac > 1 is expected and is not a measurement error; smem_bound below "
                 "is the ceiling of the algorithm actually run"),
        "smem_bound": {"achieved_GBps": lookup_bytes / (per_launch_ms * 1e-3) / 1e9,
                       "peak_GBps": peaks["smem_bytes_per_s"] / 1e9,
                       "frac": lookup_bytes / (per_launch_ms * 1e-3) / peaks["smem_bytes_per_s"],
                       "lookup_bytes_per_launch": lookup_bytes},
        "hbm": {"achieved_GBps": hbm_bytes / (per_launch_ms * 1e-3) / 1e9, "peak_GBps": hbm_peak,
                "peak_source": peak_src, "frac": hbm_bytes / (per_launch_ms * 1e-3) / 1e9 / hbm_peak,
                "bytes_per_launch": hbm_bytes},
        "traffic_source": "profiles/r0N_traffic_<kernel>.json (ncu dram__bytes_read+write of this kernel "
                          "on this workload; algorithmic bytes per launch = hbm.bytes_per_launch)",
        "kernel_share_of_step": (scan_ms / args.steps) / ms_per_step,
    }

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            rate, threads, desc, kind, one = cpu_reference_sample(target_s=15.0)
            cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": kind, "sample": desc,
                   "single_thread_value": one,
                   "single_thread_sample": "4 of the config-4 requests, one thread (answer_batch as shipped)"}
        except Exception as ex:  # the oracle is optional on the measuring host
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {ex!r}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic (DetRng(3) store, DetRng(3) seeds -> ChaCha20 query vectors, SURVEY.md §8(d))",
            "config": workload_config(B),
            "parallelism": f"bucket-range shards x{world}",
            "reduce": ("none" if sh is None else
                       "fused peer epilogue (tile fix-up)" if sh.fused else "IPC xor reduce-scatter"),
            "parity": parity,
            **({"peer_bytes": peer_bytes} if peer_bytes else {}),
            "effective_scan_GBps": B * N_BUCKETS * BUCKET_BYTES / (ms_per_step * 1e-3) / 1e9,
            "gpu_launches": launches,
            "roofline": roof,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "clocks": clk.summary(),
            **({"validation_only": f"{world} ranks share {ndev} GPU(s) over gloo; timings are not scaling "
                                   "numbers"} if shared_gpu else {}),
            "peaks_measured": peaks,
        }
        print(json.dumps(line), flush=True)
    if sh is not None:
        sh.close()
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
