#!/usr/bin/env python
"""Benchmark: encrypted query x entry dot products per second (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl wally|reference]

One step = one pass of the whole hot path over one batch (SURVEY.md §8(a)
rows a1-a6): the batcher, the forward NTT of every query ciphertext and the
fused pointwise-modmul / inverse-NTT / modulus-switch kernel that writes
every single-limb response ciphertext, for the configuration's full query
batch (default: configs[2] "c3", the paper-scale 3.2M-entry workload the
north star names; all inputs resident in HBM when the timed region starts).

Multi-GPU (one process per GPU; `--gpus N` without WORLD_SIZE re-launches
itself under torch.distributed.run with N ranks): clusters are owned by ranks
(greedy LPT on expected work, hot clusters replicated --
wally_assign_owners_replicated); the batch is resident on the ingress rank
0, whose cluster ids go to every rank over the gloo control group, and every
timed step scatters each owner's queries with the C ABI's NCCL data plane
(wally_scatter_queries: pack kernel + grouped ncclSend/ncclRecv) before the
owners evaluate them; value = all ranks' dot products / max-over-ranks
device time.  `--dry-run` runs the same routing and a gloo scatter on host
tensors without a GPU (the CPU test of the launch path).

`--impl reference` times the CPU oracle (oracle/, plain C) on this host's
cores on a bounded sample of the same workload (the reference arm).
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

import synth  # noqa: E402

METRIC = "encrypted query x entry dot products/sec"
UNIT = "dot products/s"
SM_COUNT = 148
# Integer roofline: the FMA-heavy pipe issues 64 IMAD
# per clock per SM (4 SMSPs x 16 lanes; B300_MICROARCH.md "Pipe rates",
# rt_SMSP = 2), and IMAD.HI occupies it for two slots (measured on B200:
# profiles/r01_intpipe_ncu.txt, 31.8 IMAD.HI vs 63.3 IMAD per clock per SM).
# A Shoup modmul is IMAD.HI + 2 IMAD = 4 slots, so the pipe peaks at 16
# modmuls per clock per SM (measured: 15.94).
IMAD_SLOTS_PER_CLK_PER_SM = 64
SLOTS_PER_MODMUL = 4
MODMUL_PER_CLK_PER_SM = IMAD_SLOTS_PER_CLK_PER_SM / SLOTS_PER_MODMUL
MEASURED_MODMUL_PER_CLK_PER_SM = 15.94   # intpipe_bench shoup_modmul under ncu


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c3", choices=sorted(synth.WORKLOADS))
    ap.add_argument("--impl", default="wally", choices=["wally", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--e2e-sub-batch", type=int, default=1024)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--quiet", action="store_true")
    ap.add_argument("--resp", default="auto", choices=["auto", "compact_drop", "compact", "full"],
                    help="response format (SURVEY 8(f)-1): compact = c0 only at the E result coefficients + c1; "
                         "compact_drop = compact with c1's 6 LSBs dropped (24-bit, n = 4096); auto = compact_drop "
                         "where allowed, else compact")
    ap.add_argument("--path", default="coeff", choices=["coeff", "simd"],
                    help="coeff: the coefficient-packed path (north star); simd: the paper's SIMD formulation "
                         "(diagonals + BSGS rotations with hybrid key switching, SURVEY 8(f)-3)")
    ap.add_argument("--queries", type=int, default=0,
                    help="profiling only: evaluate just the first Q queries of the batch (not a bench line)")
    ap.add_argument("--dry-run", action="store_true",
                    help="no GPU: ranks over gloo run the routing plan and the query scatter on host tensors "
                         "(checks the multi-rank launch path; prints a JSON line with value null)")
    return ap.parse_args()


def _free_port() -> int:
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def relaunch_if_needed(args):
    """`--gpus N` must run N ranks.  Without WORLD_SIZE (a plain `python bench.py
    --gpus N`), re-execute under torch.distributed.run with N local ranks and
    exit with its status; under a launcher, WORLD_SIZE must equal --gpus."""
    env_world = os.environ.get("WORLD_SIZE")
    if env_world is None:
        if args.gpus > 1:
            cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
                   "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__),
                   *sys.argv[1:]]
            log("launching", args.gpus, "ranks:", " ".join(cmd))
            sys.exit(subprocess.run(cmd).returncode)
        return
    if int(env_world) != args.gpus:
        print(f"bench.py: WORLD_SIZE={env_world} but --gpus {args.gpus}: the two must agree", file=sys.stderr)
        sys.exit(2)


def log(*a):
    print("[bench]", *a, file=sys.stderr, flush=True)


# ---------------------------------------------------------------------------
# workload arithmetic (counts only)
# ---------------------------------------------------------------------------

def modmul_per_pair(n: int, L: int) -> int:
    """Algorithmic modular multiplications per (query, plaintext) pair in the
    fused kernel: 2 components x [pointwise L n +
    inverse NTT L (n/2) log2 n + modulus switch n L(L-1)/2]."""
    lg = n.bit_length() - 1
    return 2 * (L * n + L * (n // 2) * lg + n * L * (L - 1) // 2)


def hbm_bytes_per_batch(w, nq, pairs, clusters_touched_pts, words_per_pt):
    """Algorithmic HBM bytes of the fused kernel for one batch: every needed
    plaintext (values + Shoup companions) read once, every query's NTT form
    read once, every response written once."""
    pt = clusters_touched_pts * w.num_limbs * 2 * w.n * 4
    q = nq * 2 * w.num_limbs * w.n * 4
    r = pairs * words_per_pt * 4
    return pt + q + r


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")] + [time.time()])

    def wait_first(self, timeout=5.0):
        t0 = time.time()
        while self.proc and not self.rows and time.time() - t0 < timeout:
            time.sleep(0.05)

    def mark(self):
        return time.time()

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self, t0=None, t1=None):
        rows = self.rows
        if t0 is not None:
            win = [r for r in rows if t0 - 0.25 <= r[-1] <= t1 + 0.25]
            rows = win if win else rows[-1:]
        self.rows = rows
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for i, nm in enumerate(names):
                if len(r) > 4 + i and r[4 + i].lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def ncu_traffic(config: str):
    """dram read+write bytes per launch of the fused kernel from a committed
    `ncu --set full` summary (profiles/), or None."""
    p = os.path.join(ROOT, "profiles", "ncu_fused_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        e = d.get(config)
        return int(e["bytes"]) if e else None
    except Exception:
        return None


# ---------------------------------------------------------------------------
# CPU oracle baseline (rank 0, N=1 only; also the --impl reference arm)
# ---------------------------------------------------------------------------

def oracle_sample(w, moduli, ents, ids, cts_host_fn, seconds: float, seed: int = 7):
    """Time the oracle (as it stands) on a bounded sample of (query, plaintext)
    pairs of this workload using every host core.  Returns a dict."""
    from oracle import capi
    E = w.n // w.d
    P = -(-w.cluster_size // E)
    rng = np.random.default_rng(seed)
    cores = len(os.sched_getaffinity(0))

    def run(npairs, threads=None):
        qsel = rng.integers(0, ids.size, size=npairs)
        ksel = rng.integers(0, P, size=npairs)
        uq, inv = np.unique(qsel, return_inverse=True)
        cts = cts_host_fn(uq)
        keys = sorted(set((int(ids[q]), int(k)) for q, k in zip(qsel, ksel)))
        pidx = {ck: i for i, ck in enumerate(keys)}
        pcs = np.stack([capi.encode_plaintext(ents[c][k * E:(k + 1) * E], w.d, w.n) for c, k in keys])
        pp = np.array([pidx[(int(ids[q]), int(k))] for q, k in zip(qsel, ksel)], dtype=np.uint32)
        dots = int(sum(min(E, w.cluster_size - int(k) * E) for k in ksel))
        t0 = time.perf_counter()
        _, used = capi.server_pairs(moduli, cts, pcs, inv.astype(np.uint32), pp, threads=threads or cores)
        dt = time.perf_counter() - t0
        return npairs, dots, dt, used

    n0, d0, t0, used = run(max(cores, 8))
    rate = n0 / t0
    npairs = max(cores, int(rate * seconds))
    n1, d1, t1, used = run(npairs)
    # the same oracle on one core, a sample of about 3 s
    n2, d2, t2, _ = run(max(4, int(rate / max(used, 1) * 3.0)), threads=1)
    return {"value": d1 / t1, "unit": UNIT, "cores": int(used), "kind": "oracle",
            "value_1core": round(d2 / t2, 2),
            "sample": f"{n1} random (query, plaintext) pairs of {w.name} ({d1} dot products) in {t1:.1f} s "
                      f"with {used} OpenMP threads; plain C oracle, uint64 % arithmetic; value_1core: {n2} pairs "
                      f"in {t2:.1f} s on one thread"}


# ---------------------------------------------------------------------------
# the product arm
# ---------------------------------------------------------------------------

def run_wally(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_2406_06761_b200.wally import WallyServer

    torch.cuda.set_device(local_rank)
    dev = f"cuda:{local_rank}"
    w = synth.WORKLOADS[args.config]
    t_setup = time.time()
    ents = synth.cluster_entries(w)
    ids_all = synth.query_clusters(w)
    C = w.num_clusters
    sizes = np.full(C, w.cluster_size, np.uint32)
    E = w.n // w.d
    P = -(-w.cluster_size // E)
    from paper_2406_06761_b200 import wally as W
    # cluster ownership (N > 1): greedy LPT on expected work = prior query share x P_c, with
    # clusters heavier than the mean rank load replicated (profiles/r01_balance.txt)
    owner = W.wally_assign_owners_replicated(synth.cluster_popularity(w) * P, world) if world > 1 else None
    if args.resp == "auto":
        args.resp = "compact_drop" if w.n == 4096 else "compact"
    fmt = {"full": W.WALLY_RESP_FULL, "compact": W.WALLY_RESP_COMPACT,
           "compact_drop": W.WALLY_RESP_COMPACT_DROP}[args.resp]
    srv = WallyServer(w.n, w.num_limbs, w.d, w.t, device=local_rank, resp_format=fmt)
    moduli = srv.moduli
    srv.load_clusters(sizes, owner, rank)
    local = srv.local_cluster_ids()
    ent_dev = torch.from_numpy(np.ascontiguousarray(ents[local]).reshape(-1, w.d)).to(dev)
    torch.cuda.synchronize()
    te = time.time()
    srv.encode(ent_dev)
    torch.cuda.synchronize()
    encode_s = time.time() - te
    del ent_dev
    nsel = args.queries if args.queries > 0 else ids_all.size
    ids_in = np.ascontiguousarray(ids_all[:nsel])
    router = None
    comm = None
    if world > 1:
        # queries arrive on the ingress rank 0 (resident in its HBM); every step
        # broadcasts their cluster ids over the gloo control plane (host tensors,
        # no device sync), routes (wally_route_plan, same on every rank) and
        # scatters each owner's share with the C ABI's NCCL data plane
        from paper_2406_06761_b200.dist import Router
        router = Router(sizes, owner, w.n, w.d, w.num_limbs, srv=srv, device=dev, transport="wally")
        comm = {"nranks": srv.comm_world, "rank": srv.comm_rank,
                "transport": "NCCL communicator inside libwally.so (wally_comm_init / wally_scatter_queries / "
                             "wally_gather_responses); control plane (cluster ids, unique id) over gloo"}
        log(f"rank {rank}: wally NCCL communicator nranks={srv.comm_world}")
        cts_in = synth.uniform_ciphertexts_torch(w, moduli, device=dev)[:nsel].contiguous() if rank == 0 else None
        plan = router.plan(ids_in)
        ids = np.ascontiguousarray(ids_in[plan.share(rank)])
        share_buf = torch.empty((max(1, int(plan.counts[rank])), 2, w.num_limbs, w.n), dtype=torch.int32,
                                device=dev)
        pack_buf = torch.empty_like(cts_in) if rank == 0 else None
        # the route order goes to the device through two pinned buffers (async copies, no stream sync)
        order_pin = [torch.empty(nsel, dtype=torch.int32).pin_memory() for _ in range(2)]
        order_dev = torch.empty(nsel, dtype=torch.int32, device=dev) if rank == 0 else None
        order_ev = [torch.cuda.Event(), torch.cuda.Event()]
        order_ev[1].record()
        step_no = [0]
    else:
        cts_in = synth.uniform_ciphertexts_torch(w, moduli, device=dev)
        if nsel < ids_all.size:
            cts_in = cts_in[:nsel].contiguous()
        ids = ids_in
    nq = int(ids.size)
    pairs = nq * P
    dots = nq * w.cluster_size
    off = srv.response_layout(ids)
    resp = torch.empty(max(1, int(off[-1])), dtype=torch.int32, device=dev)
    ws = srv.alloc_workspace(max(nq, 1))
    torch.cuda.synchronize()
    setup_s = time.time() - t_setup
    stream = torch.cuda.current_stream()

    def step():
        if router is None:
            srv.eval_batch(ids, cts_in, resp, ws)
            return cts_in
        ids_r = router.broadcast_ids(ids_in if rank == 0 else None, nsel)
        pl = router.plan(ids_r)
        if rank == 0:
            k = step_no[0] & 1
            order_ev[k].synchronize()          # the copy out of this buffer two steps ago is done
            order_pin[k].numpy()[:] = pl.order.view(np.int32)
            order_dev.copy_(order_pin[k], non_blocking=True)
            order_ev[k].record()
            step_no[0] += 1
        mine = router.scatter(pl, cts_in, out=share_buf, pack_buf=pack_buf, order_dev=order_dev)
        srv.eval_batch(ids_r[pl.share(rank)], mine, resp, ws)
        return mine

    for _ in range(args.warmup):
        cts = step()
    srv.check_batch(ws)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    srv.enable_stage_timing(True)
    srv.stage_times()
    launches0 = srv.kernel_launches()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    with ClockSampler(local_rank) as clk:
        clk.wait_first()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t_clk0 = clk.mark()
        evs[0].record(stream)
        for i in range(args.steps):
            cts = step()
            evs[i + 1].record(stream)
        torch.cuda.synchronize()
        t_clk1 = clk.mark()
    if world > 1:
        dist.barrier()
    step_ms = [evs[i].elapsed_time(evs[i + 1]) for i in range(args.steps)]
    ms = evs[0].elapsed_time(evs[-1])
    launches = srv.kernel_launches() - launches0
    st_batcher, st_fwd, st_fused, nb = srv.stage_times()
    srv.enable_stage_timing(False)
    srv.check_batch(ws)
    if router is not None:
        srv.comm_check()
    gather_ms = None
    if router is not None:
        # optional response gather to the ingress, timed separately
        ge0, ge1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        dist.barrier()
        ge0.record(stream)
        gathered = router.gather(router.plan(ids_in), resp)
        ge1.record(stream)
        torch.cuda.synchronize()
        gather_ms = ge0.elapsed_time(ge1)
        del gathered

    # max over ranks (time, per step too) and sums (work)
    t = torch.tensor([ms, st_fused / max(nb, 1), gather_ms or 0.0, *step_ms], dtype=torch.float64, device=dev)
    wk = torch.tensor([dots, pairs, nq], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(wk, op=dist.ReduceOp.SUM)
    ms_max, fused_ms_max, gather_ms_max = float(t[0]), float(t[1]), float(t[2])
    step_ms_max = [float(x) for x in t[3:]]
    tot_dots, tot_pairs, tot_nq = (int(x) for x in wk.tolist())
    ms_per_step = ms_max / args.steps
    value = tot_dots / (ms_per_step / 1e3)

    # roofline of the dominant (fused) kernel: the integer multiply (FMA-heavy) pipe
    peaks = measured_peaks()
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    clocks = clk.summary(t_clk0, t_clk1)
    mm = srv.modmuls_per_pair()                   # of the kernel variant this context runs
    mm_full = modmul_per_pair(w.n, w.num_limbs)
    modmul_per_launch = float(mm) * pairs          # this rank's launch
    fused_ms = st_fused / max(nb, 1)
    achieved = modmul_per_launch / (fused_ms / 1e3) / 1e12
    peak = SM_COUNT * MODMUL_PER_CLK_PER_SM * sm_max * 1e6 / 1e12
    sm_now = clocks.get("sm_mhz") or sm_max
    roofline = {"bound": "fmaheavy", "bound_class": "alu (integer multiply-add on the FMA-heavy pipe; no "
                                                    "tensor-core or HBM bound, DESIGN.md section 6)",
                "achieved": round(achieved, 4), "peak": round(peak, 4), "unit": "Tmodmul/s",
                "frac": round(achieved / peak, 4), "traffic": ncu_traffic(args.config),
                "frac_at_measured_clock": round(achieved / (peak * sm_now / sm_max), 4),
                "frac_vs_microbench": round(achieved / (SM_COUNT * MEASURED_MODMUL_PER_CLK_PER_SM * sm_max * 1e6 / 1e12),
                                            4),
                "frac_vs_3imad_model": round(achieved * 3 / (SM_COUNT * 64 * sm_max * 1e6 / 1e12), 4),
                "modmul_per_pair": int(mm), "modmul_per_pair_unpruned": int(mm_full),
                "frac_unpruned_equiv": round(mm_full * pairs / (fused_ms / 1e3) / 1e12 / peak, 4),
                "kernel": "eval_kernel (fused pointwise Shoup modmul + inverse NTT + RNS mod-switch)",
                "per_launch": f"{pairs} pairs x {mm} modmul (wally_modmuls_per_pair: SURVEY.md 8(d) M_pair"
                              f"{', c0 pruned to the result coefficients' if mm < mm_full else ''})",
                "peak_basis": f"{SM_COUNT} SMs x {MODMUL_PER_CLK_PER_SM:.0f} Shoup modmul/clk/SM (64 FMA-heavy IMAD "
                              f"slots/clk/SM, IMAD.HI = 2 slots, measured) x {sm_max:.0f} MHz (sm_max_mhz of "
                              "MEASURED_PEAKS.json)",
                "fused_ms_per_launch": round(fused_ms, 4),
                "hbm_algorithmic_GBps": round(hbm_bytes_per_batch(w, nq, pairs, len(np.unique(ids)) * P,
                                                                  srv.words_per_plaintext)
                                              / (fused_ms / 1e3) / 1e9, 1),
                "hbm_peak_GBps": peaks.get("hbm_gbs")}

    out = {"metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
           "ms_per_step_best": round(min(step_ms_max), 4),
           "ms_per_step_median": round(float(np.median(step_ms_max)), 4),
           "value_best": round(tot_dots / (min(step_ms_max) / 1e3), 1),
           "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "u32",
           "data": "synthetic (seeded numpy/torch; entries per BASELINE config; query ciphertexts are uniform "
                   "RNS residues, which RLWE makes indistinguishable from fresh encryptions)",
           "config": {"workload": w.name, "description": w.description, "n": w.n, "limbs": w.num_limbs,
                      "d": w.d, "t": w.t, "clusters": w.num_clusters, "cluster_size": w.cluster_size,
                      "queries": int(tot_nq), "pairs_per_step": int(tot_pairs), "dots_per_step": int(tot_dots),
                      "response_format": f"{args.resp} ({srv.words_per_plaintext} words per plaintext; "
                                         "include/wally.h WALLY_RESP_*)",
                      "ownership": ("greedy LPT on expected work with hot-cluster replication "
                                    "(wally_assign_owners_replicated); queries resident on rank 0, scattered by "
                                    "the C ABI's NCCL data plane inside every step") if world > 1 else "single rank",
                      "l2": "inputs larger than L2 (plaintext store, query NTTs and responses >> 126 MB)"},
           "roofline": roofline,
           "stages_ms_per_step": {"batcher": round(st_batcher / max(nb, 1), 4),
                                  "forward_ntt": round(st_fwd / max(nb, 1), 4),
                                  "fused": round(fused_ms, 4)},
           "gpu_launches": int(launches),
           "comm": comm,
           "gather_ms_per_batch": round(gather_ms_max, 3) if world > 1 else None,
           "clocks": clocks,
           "setup_s": round(setup_s, 1), "encode_s": round(encode_s, 3)}
    if args.queries > 0:
        out["profiling_subset"] = f"first {args.queries} queries only -- not a bench line"

    # end-to-end through the host-buffer C-ABI call (pinned host memory)
    if not args.no_e2e and args.e2e_steps > 0:
        try:
            out["e2e"] = run_e2e(args, srv, ids, cts, off, world, rank, local_rank, dots)
        except Exception as e:  # report, never hide
            out["e2e"] = {"value": None, "unit": UNIT, "error": repr(e)[:300]}
    del resp, ws
    torch.cuda.empty_cache()

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        def cts_host(qidx):
            return cts[torch.from_numpy(qidx).to(dev)].cpu().numpy().view(np.uint32)
        out["cpu_baseline"] = oracle_sample(w, moduli, ents, ids, cts_host, args.cpu_seconds)
    srv.close()
    return out


def run_e2e(args, srv, ids, cts, off, world, rank, local_rank, dots_local):
    import torch
    import torch.distributed as dist
    dev = f"cuda:{local_rank}"
    words = int(off[-1])
    qh = torch.empty(cts.shape, dtype=torch.int32, pin_memory=True)
    qh.copy_(cts)
    rh = torch.empty(words, dtype=torch.int32, pin_memory=True)
    sub = args.e2e_sub_batch
    ws = torch.empty(srv.host_workspace_bytes(sub) // 4 + 64, dtype=torch.int32, device=dev)
    srv.eval_batch_host(ids, qh, rh, sub, ws)  # warm-up
    stream = torch.cuda.current_stream()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    start.record(stream)
    for _ in range(args.e2e_steps):
        srv.eval_batch_host(ids, qh, rh, sub, ws)
    end.record(stream)
    torch.cuda.synchronize()
    ms = start.elapsed_time(end) / args.e2e_steps
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    d = torch.tensor([dots_local], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(d, op=dist.ReduceOp.SUM)
    h2d = int(cts.numel() * 4)
    d2h = int(words * 4)
    del ws, qh, rh
    return {"value": round(float(d[0]) / (float(t[0]) / 1e3), 1), "unit": UNIT,
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": round(float(t[0]), 3),
            "api": "wally_eval_batch_host (pinned host query ciphertexts -> device -> pinned host responses, "
                   f"sub-batches of {sub} queries overlapped on two streams)", "steps": args.e2e_steps}


# ---------------------------------------------------------------------------
# the SIMD formulation: a second bench line, not the default
# ---------------------------------------------------------------------------

def run_simd(args, rank, world, local_rank):
    """One step = wally_simd_eval_batch over the configuration's query batch:
    NTT of every query ciphertext and both rotation keys, g - 1 baby-step
    rotations per query, the diagonal inner products, m - 1 giant-step
    rotations and the switch to q_0 per (query, block).  Ranks > 1 run
    independent replicas on disjoint query shares (no collective: the SIMD
    path shards by query like the coefficient path)."""
    import torch
    import torch.distributed as dist
    from paper_2406_06761_b200.simd import STAGES as STAGES_SIMD, SimdServer

    torch.cuda.set_device(local_rank)
    dev = f"cuda:{local_rank}"
    w = synth.WORKLOADS[args.config]
    t_setup = time.time()
    ents = synth.cluster_entries(w)
    ids_all = synth.query_clusters(w)
    srv = SimdServer(w.n, w.num_limbs, w.d, w.t, device=local_rank)
    te = time.time()
    srv.load_clusters([ents[c] for c in range(w.num_clusters)])
    torch.cuda.synchronize()
    encode_s = time.time() - te
    nsel = args.queries if args.queries > 0 else ids_all.size
    share = np.arange(nsel)[rank::world]
    ids = np.ascontiguousarray(ids_all[share])
    nq = int(ids.size)
    cts = synth.uniform_ciphertexts_torch(w, srv.moduli[:w.num_limbs], device=dev)[:nsel]
    keys = synth.uniform_keys_torch(w, srv.moduli, num_queries=nsel, device=dev)
    if world > 1:
        sel = torch.from_numpy(share).to(dev)
        cts, keys = cts[sel].contiguous(), keys[sel].contiguous()
    cts = cts.contiguous()
    words = srv.response_words(ids)
    resp = torch.empty(max(1, words), dtype=torch.int32, device=dev)
    blocks = np.array([srv.blocks(int(c)) for c in ids])
    dots = nq * w.cluster_size
    torch.cuda.synchronize()
    setup_s = time.time() - t_setup
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        srv.eval_batch(ids, cts, keys, resp)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches0 = srv.launch_count()
    srv.stage_times()                                  # clear
    srv.enable_stage_timing(True)
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        clk.wait_first()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t_clk0 = clk.mark()
        start.record(stream)
        for _ in range(args.steps):
            srv.eval_batch(ids, cts, keys, resp)
        end.record(stream)
        torch.cuda.synchronize()
        t_clk1 = clk.mark()
    ms = start.elapsed_time(end)
    srv.enable_stage_timing(False)
    st_ms, _ = srv.stage_times()
    launches = srv.launch_count() - launches0
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    wk = torch.tensor([dots, nq], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(wk, op=dist.ReduceOp.SUM)
    ms_per_step = float(t[0]) / args.steps
    tot_dots, tot_nq = (int(x) for x in wk.tolist())
    value = tot_dots / (ms_per_step / 1e3)
    peaks = measured_peaks()
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    clocks = clk.summary(t_clk0, t_clk1)
    mm = sum(srv.modmuls_per_query(int(b)) for b in blocks)
    peak = SM_COUNT * MODMUL_PER_CLK_PER_SM * sm_max * 1e6 / 1e12
    hbm_peak = float(peaks.get("hbm_gbs", 6556.5))
    # per-stage roofline (include/wally_simd.h wally_simd_stage_work): each stage is bound by the larger of
    # its modmuls on the integer pipe and its minimum HBM bytes; the step's bound is their sum
    smm, sby = srv.stage_work(ids)
    stages, t_bound = {}, 0.0
    for i, name in enumerate(STAGES_SIMD):
        sms = st_ms[i] / args.steps
        t_int = smm[i] / (peak * 1e12) * 1e3
        t_hbm = sby[i] / (hbm_peak * 1e9) * 1e3
        tb = max(t_int, t_hbm)
        t_bound += tb
        stages[name] = {"ms": round(sms, 3), "modmuls": smm[i], "bytes": sby[i],
                        "bound": "fmaheavy" if t_int >= t_hbm else "hbm",
                        "achieved": round(smm[i] / (sms / 1e3) / 1e12, 4) if t_int >= t_hbm
                        else round(sby[i] / (sms / 1e3) / 1e9, 1),
                        "unit": "Tmodmul/s" if t_int >= t_hbm else "GB/s",
                        "frac": round(tb / sms, 4) if sms > 0 else None}
    rot_ms = (st_ms[1] + st_ms[3]) / args.steps
    rot_mm = smm[1] + smm[3]
    achieved = rot_mm / (rot_ms / 1e3) / 1e12
    roofline = {"bound": "fmaheavy", "bound_class": "alu (integer multiply-add on the FMA-heavy pipe, DESIGN.md "
                                                    "section 6)",
                "achieved": round(achieved, 4), "peak": round(peak, 4), "unit": "Tmodmul/s",
                "frac": round(achieved / peak, 4), "traffic": None,
                "kernel": "the rotations (baby and giant steps: simd_rot_chain_kernel, or simd_modup/moddown), "
                          f"{100 * rot_ms / (ms / args.steps):.0f}% of the step, timed by the library's stage events",
                "per_launch": f"{rot_mm} modmul per step in the rotations (wally_simd_stage_work)",
                "peak_basis": f"{SM_COUNT} SMs x {MODMUL_PER_CLK_PER_SM:.0f} Shoup modmul/clk/SM x {sm_max:.0f} MHz",
                "step_frac": round(t_bound / (ms / args.steps), 4),
                "step_bound_ms": round(t_bound, 3),
                "step_frac_basis": "sum over the five stages of max(modmuls / integer peak, bytes / HBM peak "
                                   f"{hbm_peak:.0f} GB/s) divided by the measured step time",
                "frac_all_int_pipe": round(mm / (ms / args.steps / 1e3) / 1e12 / peak, 4),
                "stages": stages}
    out = {"metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "u32",
           "data": "synthetic (seeded; query ciphertexts and rotation keys are uniform RNS residues)",
           "path": "simd (SURVEY.md 8(f)-3: diagonal packing + BSGS rotations, hybrid key switching)",
           "config": {"workload": w.name + "-simd", "description": w.description, "n": w.n, "limbs": w.num_limbs,
                      "special_prime": srv.moduli[-1], "d": w.d, "t": w.t, "baby": srv.baby, "giant": srv.giant,
                      "row_slices": srv.row_slices, "block_entries": srv.block_entries,
                      "queries": int(tot_nq), "blocks_per_step": int(blocks.sum()), "dots_per_step": int(tot_dots),
                      "key_bytes_per_query": int(srv.key_words * 4),
                      "l2": "inputs larger than L2 (plaintexts, keys and ciphertexts >> 126 MB)"},
           "roofline": roofline, "gpu_launches": int(launches), "clocks": clocks,
           "setup_s": round(setup_s, 1), "encode_s": round(encode_s, 3)}
    if args.queries > 0:
        out["profiling_subset"] = f"first {args.queries} queries only -- not a bench line"
    if not args.no_e2e and args.e2e_steps > 0:
        # end to end through wally_simd_eval_batch_host: pinned host ciphertexts + keys in, responses out,
        # sub-batches pipelined (copies overlap the computation)
        qh = torch.empty(cts.shape, dtype=torch.int32, pin_memory=True)
        qh.copy_(cts)
        kh = torch.empty(keys.shape, dtype=torch.int32, pin_memory=True)
        kh.copy_(keys)
        rh = torch.empty(resp.numel(), dtype=torch.int32, pin_memory=True)
        sub = args.e2e_sub_batch
        srv.eval_batch_host(ids, qh, kh, rh, sub)          # warm-up
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.e2e_steps):
            srv.eval_batch_host(ids, qh, kh, rh, sub)
        e1.record(stream)
        torch.cuda.synchronize()
        ems = e0.elapsed_time(e1) / args.e2e_steps
        out["e2e"] = {"value": round(dots / (ems / 1e3), 1), "unit": UNIT,
                      "h2d_bytes_per_step": int((cts.numel() + keys.numel()) * 4), "d2h_bytes_per_step": int(words * 4),
                      "ms_per_step": round(ems, 3), "steps": args.e2e_steps,
                      "api": "wally_simd_eval_batch_host (pinned host ciphertexts and keys -> device -> pinned host "
                             f"responses, sub-batches of {sub} queries, copies overlapped with the computation)"}
        del qh, kh, rh
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = simd_oracle_sample(w, srv, ents, ids, cts, keys)
    srv.close()
    return out


def simd_oracle_sample(w, srv, ents, ids, cts, keys, nsample: int = 1):
    """The SIMD oracle (oracle/wally_simd_oracle.c, single thread) timed on
    `nsample` queries of the batch: its BSGS server computation and q_0
    switch; the plaintext encoding (offline ServerInit) is not timed."""
    from oracle import capi
    mods = np.array(srv.moduli, dtype=np.uint32)
    per = srv.block_entries
    tot_t, tot_dots = 0.0, 0
    for qi in range(nsample):
        c = int(ids[qi])
        ct = cts[qi].cpu().numpy().view(np.uint32)
        key = keys[qi].cpu().numpy().view(np.uint32)
        for b in range(-(-w.cluster_size // per)):
            blk = ents[c][b * per:(b + 1) * per]
            pt = np.stack([capi.simd_encode(x, w.t) for x in capi.simd_diagonal_slots(blk, w.n, w.t, w.d, srv.baby)])
            t0 = time.perf_counter()
            res = capi.simd_server(mods, w.t, w.d, srv.baby, ct, key[0], key[1], pt)
            capi.simd_response(mods[:w.num_limbs], res)
            tot_t += time.perf_counter() - t0
            tot_dots += blk.shape[0]
    return {"value": round(tot_dots / tot_t, 2), "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"{nsample} query of {w.name}-simd ({tot_dots} dot products) in {tot_t:.1f} s: the plain C "
                      "SIMD oracle (BSGS server + q_0 switch, single thread); plaintext encoding not timed"}


# ---------------------------------------------------------------------------
# the reference arm: the CPU oracle as it stands
# ---------------------------------------------------------------------------

def run_reference(args):
    from oracle import capi
    w = synth.WORKLOADS[args.config]
    moduli = capi.find_primes(w.n, w.num_limbs)
    ents = synth.cluster_entries(w)
    ids = synth.query_clusters(w)
    E = w.n // w.d
    P = -(-w.cluster_size // E)
    cores = len(os.sched_getaffinity(0))
    rng = np.random.default_rng(11)
    # one fixed sample of pairs per step, sized for ~3 s of oracle work: the plain
    # oracle takes ~11 ms per c3 pair per core (profiles/r01_bench_c3_final.json cpu_baseline)
    per_core = {"c1": 400, "c2": 270, "c3": 270, "c4": 90, "c5": 400}.get(w.name, 200)
    npairs = max(cores, per_core * cores)
    qsel = rng.integers(0, ids.size, size=npairs)
    ksel = rng.integers(0, P, size=npairs)
    uq, inv = np.unique(qsel, return_inverse=True)
    cts = synth.uniform_ciphertexts(synth.scaled(w, num_queries=len(uq)), moduli)
    keys = sorted(set((int(ids[q]), int(k)) for q, k in zip(qsel, ksel)))
    pidx = {ck: i for i, ck in enumerate(keys)}
    pcs = np.stack([capi.encode_plaintext(ents[c][k * E:(k + 1) * E], w.d, w.n) for c, k in keys])
    pp = np.array([pidx[(int(ids[q]), int(k))] for q, k in zip(qsel, ksel)], dtype=np.uint32)
    dots = int(sum(min(E, w.cluster_size - int(k) * E) for k in ksel))
    used = cores
    for _ in range(args.warmup):
        _, used = capi.server_pairs(moduli, cts, pcs, inv.astype(np.uint32), pp, threads=cores)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        _, used = capi.server_pairs(moduli, cts, pcs, inv.astype(np.uint32), pp, threads=cores)
    dt = (time.perf_counter() - t0) / args.steps
    value = dots / dt
    sample = (f"{npairs} random (query, plaintext) pairs of {w.name} per step ({dots} dot products); "
              f"plain C oracle with {used} OpenMP threads")
    return {"metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(dt * 1e3, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u64 (oracle % arithmetic)",
            "data": "synthetic (seeded)", "impl": "reference",
            "config": {"workload": w.name, "description": w.description},
            "cpu_baseline": {"value": round(value, 1), "unit": UNIT, "cores": int(used), "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": round(value, 1), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def run_dry(args, rank, world):
    """The multi-rank launch path without a GPU (gloo, host tensors): the
    ownership map, the ingress's cluster-id broadcast, the routing plan and
    the query scatter of a 512-query slice of the configuration, each share
    checked against the plan.  No CUDA call is made; value is null."""
    import torch
    from paper_2406_06761_b200 import wally as W
    from paper_2406_06761_b200.dist import Router
    w0 = synth.WORKLOADS[args.config]
    w = synth.scaled(w0, num_queries=min(w0.num_queries, 512))
    E = w.n // w.d
    P = -(-w.cluster_size // E)
    sizes = np.full(w.num_clusters, w.cluster_size, np.uint32)
    owner = W.wally_assign_owners_replicated(synth.cluster_popularity(w) * P, world)
    ids_in = synth.query_clusters(w)
    moduli = W.wally_find_moduli(w.n, w.num_limbs)
    cts = torch.from_numpy(synth.uniform_ciphertexts(w, moduli).view(np.int32)) if rank == 0 else None
    rt = Router(sizes, owner, w.n, w.d, w.num_limbs,
                pack=lambda idx, c: c[torch.from_numpy(idx.astype(np.int64))].contiguous())
    t0 = time.perf_counter()
    counts = None
    for _ in range(max(1, args.steps)):
        ids = rt.broadcast_ids(ids_in if rank == 0 else None, ids_in.size)
        assert np.array_equal(ids, ids_in)
        plan = rt.plan(ids)
        share = rt.scatter(plan, cts)
        assert share.shape[0] == int(plan.counts[rank])
        counts = plan.counts.tolist()
    dt = time.perf_counter() - t0
    return {"metric": METRIC, "value": None, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(dt * 1e3 / max(1, args.steps), 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic (seeded)",
            "dry_run": "gloo on host tensors, no GPU: ownership, id broadcast, routing plan and query scatter only",
            "config": {"workload": w0.name, "queries": int(w.num_queries), "routed_counts": counts}}


def main():
    args = parse()
    if not (args.impl == "reference" and "WORLD_SIZE" not in os.environ):
        relaunch_if_needed(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        # the oracle arm: rank 0 alone runs and prints; the other ranks exit without work
        if rank == 0:
            print(json.dumps(run_reference(args)), flush=True)
        return
    import torch
    import torch.distributed as dist
    if args.dry_run:
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", str(_free_port()))
            dist.init_process_group("gloo", rank=0, world_size=1)
        else:
            dist.init_process_group("gloo")
        out = run_dry(args, rank, world)
    else:
        if world > 1:
            torch.cuda.set_device(local_rank)
            # host tensors (cluster ids, the NCCL unique id) over gloo, device tensors over NCCL
            dist.init_process_group("cpu:gloo,cuda:nccl", device_id=torch.device(f"cuda:{local_rank}"))
        out = run_simd(args, rank, world, local_rank) if args.path == "simd" else run_wally(args, rank, world,
                                                                                            local_rank)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if dist.is_initialized():
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
