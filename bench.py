"""Benchmark of the DESSERT vector-set search hot path on B200 (driver contract: one JSON line).

Default workload (BASELINE.json configs[4], "cfg4" -- the largest single-GPU
config, on which the north star's 8M-set target is quoted): N = 8,000,000 sets,
m_i = clip(round(N(70, 25)), 8, 180) (~560 M vectors), codes only in HBM
(L = 32 tables x C = 8 bits = 32 B per vector, 17.9 GB of plane records),
generated on the GPU by hashing unit mixture vectors over 262,144 centroids;
1,024 query sets of m_q = 32 fp16 vectors; exhaustive scoring of every set;
top-1,000 per query set.
A step = hash the 32,768 query vectors (K1, tcgen05) + score every (query
set, set) pair and keep the top-1,000 (dsrt_search_all: K3 with the
threshold-append epilogue + K4 merges; no score matrix in HBM), inputs
resident in HBM.  17.9 GB of records >> 126 MB L2: no flush needed.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--config 1|2|3|4]

--config 1 / 2 / 3 run the other BASELINE configs (cfg1 exhaustive 100k sets,
cfg2 index build, cfg3 prefilter pipeline); their lines are kept in profiles/.

Multi-GPU (torchrun, --config 4): ONE index sharded by shard_bounds (contiguous
set ranges, equal vector counts; strong scaling), every rank scores its shard,
local top-k all-gathered over NCCL and merged on the device with the same
(score desc, doc id asc) key; rank 0 checks the merged top-k of 8 query sets
against the unsharded index.

--impl reference: the unmodified reference package (baseline/_ref) through its
public build_index / query API on the host cores (bench_reference.py), on a
bounded sample of the same workload; rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

UNIT = "set-pairs/s"
SPECS = {
    # workload -> (metric, L, C, size_sd, n_centroids, top_k, n_qsets, n_sets)
    4: ("set-pair scores/sec (cfg4: 8M sets x 1024 query sets, L=32 C=8, exhaustive, top-1000)",
        32, 8, 25.0, 262_144, 1000, 1024, 8_000_000),
    1: ("set-pair scores/sec (cfg1: 100k sets x 1000 query sets, L=64 C=7, exhaustive, top-100)",
        64, 7, 20.0, 4096, 100, 1000, 100_000),
}


def _dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _peaks():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            p = json.load(f)
        return p, "MEASURED_PEAKS.json"
    except (OSError, ValueError):
        return {"bf16_tflops": 1590.0, "hbm_gbs": 6650.0}, "B200_PROFILING.md fallback"


def _ncu_traffic(config: str, scale: float = 1.0):
    """Per-launch DRAM bytes (read + write) of the dominant kernel from the committed
    `ncu --set full` capture (profiles/r02_ncu_traffic.json, else r01), scaled to a launch."""
    for name in ("r02_ncu_traffic.json", "r01_ncu_traffic.json"):
        path = os.path.join(REPO, "profiles", name)
        try:
            with open(path) as f:
                rec = json.load(f)[config]
        except (OSError, KeyError, ValueError):
            continue
        return rec["traffic_bytes"] * scale, {"source": f"profiles/{name} (" + rec["source"] + ")",
                                              "captured_launch": rec["launch"],
                                              "dram_read_bytes": rec["dram_read_bytes"] * scale,
                                              "dram_write_bytes": rec["dram_write_bytes"] * scale}
    return None, None


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock + clock-event reasons sampled DURING the timed region.

    NVML (nvidia-ml-py) polled from a thread every ~2 ms, so even a 10 ms timed
    region gets samples; start() returns after the first sample.  Falls back to
    `nvidia-smi -lms 100` when NVML is unavailable.  Samples are also written to
    gpurun_out/clocks_rank<i>.csv."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.path = os.path.join(REPO, "gpurun_out", f"clocks_rank{gpu_index}.csv")
        self.samples = []
        self.thread = None
        self.proc = None

    def _handle(self, nv):
        try:
            import torch

            p = torch.cuda.get_device_properties(self.gpu)
            bus = f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
            return nv.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            return nv.nvmlDeviceGetHandleByIndex(self.gpu)

    def start(self):
        import threading

        try:
            import pynvml as nv

            nv.nvmlInit()
            h = self._handle(nv)
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            self.stop_evt = threading.Event()
            first = threading.Event()

            def loop():
                while not self.stop_evt.is_set():
                    try:
                        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                        rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.samples.append((time.perf_counter(), sm, mx, rs))
                    except Exception:
                        pass
                    first.set()
                    time.sleep(0.002)

            self.thread = threading.Thread(target=loop, daemon=True)
            self.thread.start()
            first.wait(1.0)
            return
        except Exception:
            self.thread = None
        try:
            os.makedirs(os.path.dirname(self.path), exist_ok=True)
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.fh,
                stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.thread is not None:
            self.stop_evt.set()
            self.thread.join(timeout=5)
            sm = [s[1] for s in self.samples]
            mx = [s[2] for s in self.samples]
            reasons = sorted({nm for s in self.samples for nm, bit in self.REASONS.items() if s[3] & bit})
            try:
                os.makedirs(os.path.dirname(self.path), exist_ok=True)
                with open(self.path, "w") as fh:
                    fh.write("t_s,sm_mhz,sm_max_mhz,reasons_mask\n")
                    for t, a, b, r in self.samples:
                        fh.write(f"{t:.4f},{a},{b},{r:#x}\n")
            except Exception:
                pass
            return {"sm_mhz": float(np.median(sm)) if sm else None,
                    "sm_max_mhz": float(max(mx)) if mx else None, "reasons": reasons,
                    "samples": len(sm), "source": "nvml, 2 ms poll"}
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.fh.close()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": float(max(mx)) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm), "source": "nvidia-smi -lms 100"}


# ------------------------------------------------------------------ helpers
def _timed(step_fn, steps, warmup, local, stream, world=1):
    """W untimed warm-up steps; then K steps bracketed by barrier + synchronize, timed
    with CUDA events on the launch stream; max over ranks; clocks sampled meanwhile."""
    import torch
    import torch.distributed as dist

    if os.environ.get("DSRT_PROFILE_STEPS"):  # ncu --profile-from-start off: capture the steps only
        torch.cuda.cudart().cudaProfilerStart()
    for _ in range(warmup):
        step_fn(False)
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(steps):
        step_fn(True)
    t1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    if os.environ.get("DSRT_PROFILE_STEPS"):
        torch.cuda.cudart().cudaProfilerStop()
    ms = t0.elapsed_time(t1) / steps
    if world > 1:
        tt = torch.tensor([ms], device=torch.device("cuda", local))
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    return ms, clk


def hash_flip_rate(family, Q2, L, C, mode):
    """Product-path query hash bits (K1 in `mode`) vs the float64 oracle hash_matrix
    (lsh.py:90-106): flips inside / outside the |w.x| < 1e-4 |w||x| band."""
    import torch

    from oracle import dessert_oracle as O
    from paper_2210_15748_b200 import engine

    planes = family.device_planes(mode, Q2.device)
    codes, _, _ = engine.hash_vectors(Q2, planes, mode, L, C, want_records=False, check_zero=False)
    got = codes.cpu().numpy().astype(np.int64)
    X = Q2.double().cpu().numpy()
    want = O.hash_matrix(family.planes, L, C, X)
    proj = O.projections(family.planes, X)
    band = np.abs(proj) < 1e-4 * np.linalg.norm(family.planes, axis=1)[None, :] * \
        np.linalg.norm(X, axis=1)[:, None]
    bg = ((got[:, :, None] >> np.arange(C)) & 1).reshape(len(X), L * C)
    bw = ((want[:, :, None] >> np.arange(C)) & 1).reshape(len(X), L * C)
    flips = bg != bw
    torch.cuda.synchronize()
    return {"vectors": int(len(X)), "bits": int(flips.size), "flips": int(flips.sum()),
            "flips_outside_band": int((flips & ~band).sum()), "band_fraction": float(band.mean()),
            "rate": float(flips.mean()), "mode": int(mode),
            "reference": "oracle float64 hash_matrix (lsh.py:90-106), same planes"}


def _cpu_scoring_baseline(workload, n_sets, n_qsets_step, steps, warmup):
    import bench_reference as BR

    _, L, C, sd, n_cent, top_k, _, _ = SPECS[workload]
    r = BR.scoring_baseline(L=L, C=C, size_sd=sd, n_centroids=n_cent, top_k=top_k, n_sets=n_sets,
                            n_qsets_step=n_qsets_step, steps=steps, warmup=warmup)
    api = ("reference dessert.build_index + dessert.query (baseline/_ref, unmodified)"
           if r["kind"] == "reference" else "oracle port of the reference algorithm")
    r["sample"] = (f"cfg{workload}-shaped host sample: {n_sets} sets x {n_qsets_step} query sets per "
                   f"step ({r['pairs_per_step']} set-pairs, median step {r['ms_per_step']:.0f} ms), "
                   f"top-{top_k}; {api}; {r['cores']}-process fork pool, one set shard per process, "
                   "shard results merged with the reference key")
    return r


# --------------------------------------------------------- scoring (cfg4/cfg1)
def run_scoring(args, workload):
    import torch
    import torch.distributed as dist

    import paper_2210_15748_b200 as d
    from paper_2210_15748_b200 import engine, workloads
    from paper_2210_15748_b200.distributed import merge_topk_device, shard_bounds

    world, rank, local = _dist()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    metric, L, C, sd, n_cent, top_k, n_q, n_sets = SPECS[workload]
    n_sets = args.sets or n_sets
    m_q = 32
    cfg = d.IndexConfig(d=128, C=C, L=L, seed=0, filter=d.FilterConfig(enabled=False))

    # ---- setup (untimed): synthetic codes generated on the GPU, one index, sharded by rank
    t_gen = time.perf_counter()
    if workload == 4:
        sizes = workloads.set_sizes(n_sets, 70, sd, seed=400)
        recs, Qv = workloads.gpu_codes_only(sizes, cfg, n_centroids=n_cent, n_qsets=n_q, m_q=m_q,
                                            seed=401, device=dev)
    else:
        sizes = workloads.set_sizes(n_sets, 70, sd, seed=100)
        off0 = workloads.offsets(sizes)
        X, _ = workloads.gpu_mixture(int(off0[-1]), n_cent, 128, 0.05, seed=200,
                                     dtype=torch.float16, device=dev)
        Qv = workloads.gpu_queries(X, off0, n_q, m_q, seed=300)
        _, recs = d.lsh.hash_device(d.sample_srp_family(128, C, L, 0), X, want_codes=False)
        del X
    off = workloads.offsets(sizes)
    torch.cuda.synchronize()
    t_gen = time.perf_counter() - t_gen
    full = None
    if world > 1:
        s0, s1 = shard_bounds(sizes, world)[rank]
        mine = recs[int(off[s0]):int(off[s1])].clone()
        if rank == 0:  # keep the unsharded index for the merged-result check
            full = d.build_from_records(recs, sizes, np.arange(n_sets), cfg)
        del recs
        idx = d.build_from_records(mine, sizes[s0:s1], np.arange(s0, s1), cfg)
    else:
        s0, s1 = 0, n_sets
        idx = d.build_from_records(recs, sizes, np.arange(n_sets), cfg)
        del recs
    Q2 = Qv.reshape(n_q * m_q, 128).contiguous()
    mode = d.lsh.default_mode(Q2.dtype, 128, C, Q2.shape[0], L)
    planes = idx.family.device_planes(mode, dev)
    stream = torch.cuda.current_stream()
    torch.cuda.synchronize()
    state = {"ovf": 0}

    def step(timed):
        _, qrecs, _ = engine.hash_vectors(Q2, planes, mode, L, C, want_codes=False, check_zero=False)
        s, i, ovf = engine.search_all(idx.records, idx.set_off, idx.doc_ids_dev, qrecs, m_q, L, C,
                                      idx.lut_dev, top_k, mode=0)
        state["last_ovf"] = ovf
        if world > 1:
            gs = [torch.empty_like(s) for _ in range(world)]
            gi = [torch.empty_like(i) for _ in range(world)]
            dist.all_gather(gs, s)
            dist.all_gather(gi, i)
            s, i = merge_topk_device(torch.cat(gs, 1), torch.cat(gi, 1), top_k)
        return s, i

    engine.search_profile(False)
    step(False)  # first call: lazy init outside the measured region
    torch.cuda.synchronize()
    engine.search_profile(True)
    engine.search_profile_read()

    ms, clk = _timed(step, args.steps, max(3, args.warmup), local, stream, world)
    prof = engine.search_profile_read()  # warm-up + timed steps
    engine.search_profile(False)
    n_prof_steps = args.steps + max(3, args.warmup)
    score_ms = prof["score_ms"] / n_prof_steps
    other_ms = prof["other_ms"] / n_prof_steps
    overflow = int(state["last_ovf"].item())
    pairs_per_step = n_q * n_sets
    value = pairs_per_step / (ms * 1e-3)

    # ---- e2e: the public API (query_batch), pinned host query vectors in, host results out
    Qh = Qv.cpu().pin_memory()
    d.query_batch(idx, Qh.to(dev, non_blocking=True), top_k, return_tensors=True)
    torch.cuda.synchronize()
    # short steps (cfg1): time ~2 s of e2e steps so clock ramps and host jitter average out
    e2e_steps = max(1, min(args.steps, max(args.e2e_steps, int(2000.0 / ms))))
    if world > 1:
        dist.barrier()
    te = time.perf_counter()
    for _ in range(e2e_steps):
        s_, i_ = d.query_batch(idx, Qh.to(dev, non_blocking=True), top_k, return_tensors=True)
        if world > 1:
            gs = [torch.empty_like(s_) for _ in range(world)]
            gi = [torch.empty_like(i_) for _ in range(world)]
            dist.all_gather(gs, s_)
            dist.all_gather(gi, i_)
            s_, i_ = merge_topk_device(torch.cat(gs, 1), torch.cat(gi, 1), top_k)
        hs, hi = s_.cpu(), i_.cpu()
    torch.cuda.synchronize()
    e2e_s = (time.perf_counter() - te) / e2e_steps
    if world > 1:
        tt = torch.tensor([e2e_s], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_s = float(tt.item())
    h2d = Qh.numel() * Qh.element_size()
    d2h = hs.numel() * 8 + hi.numel() * 8

    # ---- multi-GPU: merged top-k of 8 query sets == the unsharded index (rank 0)
    shard_check = None
    if world > 1:
        if rank == 0:
            q8 = Qv[:8].to(dev)
            ws_, wi_ = d.query_batch(full, q8, top_k, return_tensors=True)
            shard_check = {"query_sets": 8, "equal": bool(torch.equal(ws_, hs[:8].to(dev))
                                                          and torch.equal(wi_, hi[:8].to(dev)))}
        dist.barrier()

    # ---- roofline of the dominant kernel (K3 scoring launches inside dsrt_search_all)
    local_vec = int(off[s1] - off[s0])
    compares = float(n_q) * m_q * L * local_vec                    # per step, this rank
    achieved = compares / (score_ms * 1e-3)
    mb = engine.microbench_int()
    p_int = mb["lop3_ops_per_s"] * 4.0                             # 4 byte-compares / lane-op
    rec_bytes = local_vec * engine.record_words(L, C) * 4
    peaks, peaks_src = _peaks()
    # traffic: ncu capture of the last (largest) scoring launch, scaled to the whole step
    traffic, traffic_src = _ncu_traffic(f"cfg{workload}", 1.0)
    code_gbs = rec_bytes / (score_ms * 1e-3) / 1e9
    roofline = {
        "bound": "int", "unit": "Gcompare/s", "achieved": achieved / 1e9, "peak": p_int / 1e9,
        "frac": achieved / p_int, "traffic": traffic,
        "traffic_detail": dict(traffic_src or {}, algorithmic_bytes=rec_bytes,
                               ratio=None if traffic is None else traffic / rec_bytes,
                               per="one bench step (all scoring launches)"),
        "kernel": f"score_all_kernel<{C},{(L + 31) // 32},1,8,{4 if L <= 32 else 2}> (threshold-append epilogue)",
        "kernel_ms": score_ms, "other_search_ms": other_ms,
        "per_launch": {"compares": compares, "code_bytes": rec_bytes,
                       "hbm_floor_ms": rec_bytes / (peaks.get("hbm_gbs", 6650.0) * 1e9) * 1e3,
                       "note": "per step: the scoring launches of one dsrt_search_all call"},
        "achieved_hbm_gbs": code_gbs,
        "hbm_note": "code bytes of one pass over the index / scoring time; every query-set group "
                    "re-reads the records, mostly from L2 (dram traffic in traffic_detail)",
        "peak_source": "measured on this GPU in-run: LOP3 lane-ops/s x 4 (dsrt_microbench_int)",
        "int_microbench": mb,
    }
    line = {
        "metric": metric, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "u8",
        "data": f"synthetic (cfg{workload}-shaped, generated on GPU)",
        "config": {"workload": f"cfg{workload}", "n_sets": n_sets, "n_qsets": n_q, "m_q": m_q, "L": L,
                   "C": C, "top_k": top_k, "vectors": int(off[-1]), "vectors_this_rank": local_vec,
                   "l2": f"inputs larger than L2 ({rec_bytes / 1e9:.1f} GB plane records per rank), no flush",
                   "parallelism": f"shard{world} (one index, shard_bounds)" if world > 1 else "single",
                   "generation_s": t_gen},
        "query_sets_per_sec": n_q / (ms * 1e-3),
        "e2e": {"value": pairs_per_step / e2e_s, "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": e2e_s * 1e3, "steps": e2e_steps,
                "path": "query_batch (pinned host fp16 query vectors -> hash -> dsrt_search_all -> "
                        "host top-k)" + (" + NCCL all-gather + merge" if world > 1 else "")},
        "gpu_launches": int(round((1 + prof["launches"] / n_prof_steps + (1 if world > 1 else 0))
                                  * args.steps)),
        "search": {"score_ms": score_ms, "topk_and_list_ms": other_ms,
                   "launches_per_step": prof["launches"] / n_prof_steps, "overflow": overflow},
        "roofline": roofline,
        "clocks": clk,
    }
    if shard_check is not None:
        line["shard_check"] = shard_check
    if rank == 0:
        line["hash_bit_flips"] = hash_flip_rate(idx.family, Q2, L, C, mode)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        r = _cpu_scoring_baseline(workload, args.cpu_sets, 8, 2, 1)
        line["cpu_baseline"] = {"value": r["value"], "unit": UNIT, "cores": r["cores"],
                                "kind": r["kind"], "sample": r["sample"]}
    if rank == 0 and world == 1 and workload == 4 and not args.no_extra:
        # the prefilter pipeline (cfg3) measured in the same run: batch-256 query sets/s,
        # batch-1 p50/p99 through query(), e2e through query_batch (its own line, with the
        # CPU reference, comes from --config 3)
        del idx
        torch.cuda.empty_cache()
        c3 = cfg3_line(argparse.Namespace(**dict(vars(args), sets=0, steps=200, warmup=5,
                                                 no_cpu_baseline=True)))
        line["cfg3"] = {k: c3[k] for k in ("metric", "value", "unit", "ms_per_step", "batch1_latency_ms",
                                          "e2e", "kernel_ms", "clocks")}
        line["cfg3"]["roofline"] = {k: c3["roofline"][k] for k in ("bound", "kernel", "frac", "achieved", "peak", "unit")}
        del c3
        torch.cuda.empty_cache()
        # index build (cfg2): hash + layout of 10M bf16 vectors, with its sampled hash flip rate
        # 20 steps as in the driver's runs: 100 back-to-back steps of this tensor-heavy kernel
        # reach the power cap (sw_power_cap; 1.86 vs 1.62 ms per step measured)
        c2 = cfg2_line(argparse.Namespace(**dict(vars(args), vectors=0, steps=20, warmup=5,
                                                 no_cpu_baseline=True)))
        line["cfg2"] = {k: c2[k] for k in ("metric", "value", "unit", "ms_per_step", "e2e", "hash_bit_flips",
                                          "clocks")}
        line["cfg2"]["roofline"] = {k: c2["roofline"][k] for k in ("bound", "kernel", "frac", "achieved", "peak",
                                                                   "unit", "mma_frac")}
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


# ------------------------------------------------------------- reference arm
def run_reference(args):
    world, rank, _ = _dist()
    if rank != 0:
        return 0
    workload = args.config if args.config in SPECS else 4
    metric, L, C, _, _, top_k, n_q, n_sets = SPECS[workload]
    r = _cpu_scoring_baseline(workload, args.cpu_sets, 8, args.steps, args.warmup)
    v = r["value"]
    line = {
        "impl": "reference", "metric": metric, "value": v, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": r["ms_per_step"],
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
        "data": f"synthetic (cfg{workload}-shaped host sample)",
        "config": {"workload": f"cfg{workload}", "n_sets": n_sets, "n_qsets": n_q, "m_q": 32, "L": L,
                   "C": C, "top_k": top_k, "sample": f"{r['n_qsets_step']} query sets x {r['n_sets']} sets per step"},
        "step": {"measured_ms_per_step": r["ms_per_step"], "pairs_per_step": r["pairs_per_step"],
                 "full_workload_ms_extrapolated": n_q * n_sets / v * 1e3, "setup_s": r["setup_s"]},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": r["cores"], "kind": r["kind"],
                         "sample": r["sample"]},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# ------------------------------------------------------------- cfg3 / cfg2
def _clocks_and_time(step_fn, steps, warmup, local, stream):
    import torch

    if os.environ.get("DSRT_PROFILE_STEPS"):  # ncu --profile-from-start off: capture the steps only
        torch.cuda.cudart().cudaProfilerStart()
    for _ in range(warmup):
        step_fn(False)
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(steps):
        step_fn(True)
    t1.record(stream)
    torch.cuda.synchronize()
    if os.environ.get("DSRT_PROFILE_STEPS"):
        torch.cuda.cudart().cudaProfilerStop()
    return t0.elapsed_time(t1) / steps, clocks.stop()


def run_cfg3(args):
    print(json.dumps(cfg3_line(args)))
    return 0


def cfg3_line(args):
    """cfg3: 1M sets (~70M fp16 vectors) from 65,536 centroids; prefilter probe 4,
    k_filter 4,096; L=32, C=7; top-100.  Batch 256 throughput + batch-1 p50/p99."""
    import torch

    import paper_2210_15748_b200 as d
    from paper_2210_15748_b200 import _lib, engine, prefilter, workloads

    world, rank, local = _dist()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    n_sets, m_q, L, C, top_k, probe, k_filter = args.sets or 1_000_000, 32, 32, 7, 100, 4, 4096
    n_cent = 65_536
    sizes = workloads.set_sizes(n_sets, 70, 20, seed=500)
    off = workloads.offsets(sizes)
    t_gen = time.perf_counter()
    X, cents = workloads.gpu_mixture(int(off[-1]), n_cent, 128, 0.05, seed=501,
                                     dtype=torch.float16, device=dev)
    cfg = d.IndexConfig(d=128, C=C, L=L, seed=0,
                        filter=d.FilterConfig(enabled=True, centroids=n_cent, probe=probe,
                                              k_filter=k_filter))
    idx = d.build_from_vectors(X, sizes, np.arange(n_sets), cfg, keep_codes=False)
    cvec = cents.double()
    cvec = cvec / cvec.norm(dim=1, keepdim=True)
    centroids = prefilter.Centroids(k=n_cent, seed=0, vectors=cvec.cpu().numpy())
    torch.cuda.synchronize()
    t_ci = time.perf_counter()
    # exact native K6: tcgen05 screen + float64 re-rank argmax, radix counting-sort postings
    cindex = prefilter.build_centroid_index(X, centroids, set_off=idx.set_off, n_docs=n_sets)
    torch.cuda.synchronize()
    t_ci = time.perf_counter() - t_ci
    idx.filter = (centroids, cindex)
    Qall = workloads.gpu_queries(X, off, 256 + 1000, m_q, seed=502)
    del X
    torch.cuda.synchronize()
    t_gen = time.perf_counter() - t_gen
    stream = torch.cuda.current_stream()
    Qb = Qall[:256]
    kev = {"prefilter": [], "score": []}
    last = {}

    def step(timed):
        # one batch of 256 query sets through hash -> K5 -> K3 (candidates) -> K4
        Q2 = Qb.reshape(-1, 128)
        _, qrecs = d.lsh.hash_device(idx.family, Q2, want_codes=False, check_zero=False)
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)] if timed else None
        if timed:
            e[0].record(stream)
        cand, n_cand = prefilter.filter_candidates_device(cindex, centroids, Q2, m_q, probe,
                                                          k_filter)
        if timed:
            e[1].record(stream)
        scores, _ = engine.score_candidates(idx.records, idx.set_off, qrecs, m_q, L, C,
                                            idx.lut_dev, cand=cand, n_cand=n_cand)
        if timed:
            e[2].record(stream)
            kev["prefilter"].append((e[0], e[1]))
            kev["score"].append((e[1], e[2]))
        last["cand"], last["n_cand"] = cand, n_cand
        return engine.topk(scores, top_k, ids=idx.doc_ids_dev, n_valid=n_cand, id_index=cand)

    # per-stage kernel times from eager steps with events between the stages
    for _ in range(3):
        step(False)
    for _ in range(10):
        step(True)
    torch.cuda.synchronize()
    pf_ms = float(np.mean([a.elapsed_time(b) for a, b in kev["prefilter"]]))
    sc_ms = float(np.mean([a.elapsed_time(b) for a, b in kev["score"]]))
    # the batch step is a fixed sequence of ~11 kernels: capture it once in a CUDA
    # graph and time replays (no host launch gaps between the kernels)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        step(False)
    ms, clk = _clocks_and_time(lambda timed: graph.replay(), args.steps, max(3, args.warmup),
                               local, stream)
    # batch-1 latency through the public API (host query in, host results out)
    lat = []
    Qh = Qall[256:].cpu()
    for i in range(min(args.latency_queries, Qh.shape[0])):
        t = time.perf_counter()
        d.query(idx, Qh[i], top_k)
        lat.append(time.perf_counter() - t)
    lat = np.array(lat[5:]) * 1e3
    # e2e: the public batched API with host query vectors in, host results out
    Qb = Qall[:256].reshape(256, m_q, 128).cpu().pin_memory()
    for _ in range(2):
        d.query_batch(idx, Qb.to(dev, non_blocking=True), top_k, return_tensors=True)
    torch.cuda.synchronize()
    # pipelined like a serving loop: step t+1's H2D copy (side stream) and step t-1's D2H
    # read overlap step t's compute; every step still moves its own inputs and results
    n_e2e = max(5, min(args.steps, 20))
    cs, main = torch.cuda.Stream(), torch.cuda.current_stream()
    dq = [torch.empty(Qb.shape, dtype=Qb.dtype, device=dev) for _ in range(2)]
    hs = [torch.empty((256, top_k), dtype=torch.float64).pin_memory() for _ in range(2)]
    hi = [torch.empty((256, top_k), dtype=torch.int64).pin_memory() for _ in range(2)]
    h2d = [torch.cuda.Event() for _ in range(2)]
    used = [torch.cuda.Event() for _ in range(2)]
    d2h = [torch.cuda.Event() for _ in range(2)]
    torch.cuda.synchronize()
    te = time.perf_counter()
    with torch.cuda.stream(cs):
        dq[0].copy_(Qb, non_blocking=True)
        h2d[0].record(cs)
    for t in range(n_e2e):
        c = t & 1
        main.wait_event(h2d[c])
        s_, i_ = d.query_batch(idx, dq[c], top_k, return_tensors=True)
        used[c].record(main)
        if t + 1 < n_e2e:
            with torch.cuda.stream(cs):
                if t >= 1:  # the buffer's previous batch has been consumed
                    cs.wait_event(used[1 - c])
                dq[1 - c].copy_(Qb, non_blocking=True)
                h2d[1 - c].record(cs)
        hs[c].copy_(s_, non_blocking=True)
        hi[c].copy_(i_, non_blocking=True)
        d2h[c].record(main)
        if t >= 1:
            d2h[1 - c].synchronize()  # step t-1's results are on the host
    d2h[(n_e2e - 1) & 1].synchronize()
    e2e_s = (time.perf_counter() - te) / n_e2e
    hs, hi = hs[0], hi[0]
    # roofline of the dominant kernel (K3 candidate mode): compares of this batch
    sizes_dev = idx.set_off[1:] - idx.set_off[:-1]
    cnd, ncd = last["cand"], last["n_cand"]
    valid = torch.arange(cnd.shape[1], device=dev)[None, :] < ncd[:, None].long()
    cand_vec = int((sizes_dev[cnd.clamp(min=0)] * valid).sum().item())
    compares = float(cand_vec) * m_q * L
    mb = engine.microbench_int()
    p_int = mb["lop3_ops_per_s"] * 4.0
    rec_bytes = cand_vec * engine.record_words(L, C) * 4
    traffic3, t3d = _ncu_traffic("cfg3", cand_vec / 82221078.0)
    line = {
        "metric": "query sets/sec (cfg3: 1M sets, prefilter probe 4 / k_filter 4096, L=32 C=7, top-100, batch 256)",
        "value": 256 / (ms * 1e-3), "unit": "query sets/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64+u8", "data": "synthetic (cfg3-shaped, generated on GPU)",
        "config": {"workload": "cfg3", "n_sets": n_sets, "vectors": int(off[-1]), "centroids": n_cent,
                   "probe": probe, "k_filter": k_filter, "batch": 256, "top_k": top_k,
                   "setup_s": t_gen, "centroid_index_build_s": t_ci,
                   "postings": int(cindex.post_docs.shape[0])},
        "batch1_latency_ms": None if lat.size == 0 else {
            "p50": float(np.percentile(lat, 50)), "p99": float(np.percentile(lat, 99)),
            "n": int(lat.size)},
        "kernel_ms": {"prefilter": pf_ms, "score_candidates": sc_ms},
        "e2e": {"value": 256 / e2e_s, "unit": "query sets/s",
                "h2d_bytes_per_step": Qb.numel() * Qb.element_size(),
                "d2h_bytes_per_step": hs.numel() * 8 + hi.numel() * 8, "ms_per_step": e2e_s * 1e3,
                "path": "query_batch (hash -> prefilter -> candidate scoring -> top-k); pinned H2D of "
                        "the next batch and D2H of the previous results overlap the current batch"},
        "roofline": {"bound": "int", "unit": "Gcompare/s", "kernel": "score_cand_kernel<7,1,1>",
                     "kernel_ms": sc_ms, "achieved": compares / (sc_ms * 1e-3) / 1e9,
                     "peak": p_int / 1e9, "frac": compares / (sc_ms * 1e-3) / p_int,
                     "traffic": traffic3,
                     "traffic_detail": None if traffic3 is None else dict(
                         t3d, algorithmic_bytes=rec_bytes, ratio=traffic3 / rec_bytes,
                         note="candidate sets differ per query set, so every candidate's records "
                              "stream once per query set"),
                     "per_launch": {"compares": compares, "candidate_vectors": cand_vec,
                                    "code_bytes": rec_bytes,
                                    "hbm_floor_ms": rec_bytes / 6456.2e9 * 1e3},
                     "peak_source": "measured in-run: LOP3 lane-ops/s x 4"},
        "clocks": clk, "int_microbench": mb,
        # plane permute, hash, f16 rows, screen, theta, chunk candidates, re-rank, fallback,
        # count, placement plan, place, score, top-k
        "gpu_launches": 13 * args.steps,
    }
    if not args.no_cpu_baseline:
        import bench_reference as BR

        r = BR.cfg3_baseline(n_qsets=16)
        if r is not None:
            line["cpu_baseline"] = {"value": r["value"], "unit": r["unit"], "cores": r["cores"],
                                    "kind": r["kind"], "sample": r["sample"],
                                    "per_query_set_s": r["per_query_set_s"], "setup_s": r["setup_s"]}
    return line


def run_cfg2(args):
    print(json.dumps(cfg2_line(args)))
    return 0


def cfg2_line(args):
    """cfg2: index build of 10M bf16 unit vectors (cfg1 mixture, cfg1 set sizes): hash
    (tcgen05, bf16 hi/lo planes, fused sign/pack -> codes + plane records) + CSR layout."""
    import torch

    import paper_2210_15748_b200 as d
    from oracle import dessert_oracle as O
    from paper_2210_15748_b200 import _lib, engine, workloads

    world, rank, local = _dist()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    n_vec, L, C = args.vectors or 10_000_000, 64, 7
    rng = np.random.default_rng(600)
    sizes = workloads.set_sizes(int(n_vec / 60), 70, 20, seed=600)
    cs = np.cumsum(sizes)
    n_sets = int(np.searchsorted(cs, n_vec)) + 1
    sizes = sizes[:n_sets].copy()
    sizes[-1] -= int(cs[n_sets - 1] - n_vec)
    if sizes[-1] <= 0:
        sizes = sizes[:-1]
    X, _ = workloads.gpu_mixture(n_vec, 4096, 128, 0.05, seed=601, dtype=torch.bfloat16, device=dev)
    fam = d.sample_srp_family(128, C, L, 0)
    mode = _lib.HASH_TC_BF16X2
    planes = fam.device_planes(mode, dev)
    sizes_dev = torch.from_numpy(sizes).to(dev)
    stream = torch.cuda.current_stream()
    kev = []

    def step(timed):
        if timed:
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
        codes, recs, _ = engine.hash_vectors(X, planes, mode, L, C, check_zero=False)
        if timed:
            e1.record(stream)
            kev.append((e0, e1))
        set_off, _ = engine.sizes_to_offsets(sizes_dev)
        return codes, recs, set_off

    ms, clk = _clocks_and_time(step, args.steps, max(3, args.warmup), local, stream)
    k_ms = float(np.mean([a.elapsed_time(b) for a, b in kev]))
    codes, recs, set_off = step(False)
    torch.cuda.synchronize()
    # flip rate vs the float64 oracle on a sample of vectors
    samp = np.sort(rng.choice(n_vec, size=20000, replace=False))
    Xs = X[torch.from_numpy(samp).to(dev)].double().cpu().numpy()
    want = O.hash_matrix(fam.planes, L, C, Xs)
    got = codes[torch.from_numpy(samp).to(dev)].cpu().numpy().astype(np.int64)
    proj = O.projections(fam.planes, Xs)
    band = np.abs(proj) < 1e-4 * np.linalg.norm(fam.planes, axis=1)[None, :] * \
        np.linalg.norm(Xs, axis=1)[:, None]
    bg = ((got[:, :, None] >> np.arange(C)) & 1).reshape(len(samp), L * C)
    bw = ((want[:, :, None] >> np.arange(C)) & 1).reshape(len(samp), L * C)
    flips = bg != bw
    peaks = json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(REPO, "MEASURED_PEAKS.json")) else {"bf16_tflops": 1590.0, "hbm_gbs": 6650.0}
    alg_flops = 2.0 * 128 * L * C * n_vec
    mma_flops = 2 * alg_flops  # hi/lo planes: two MMA chains
    hbm_bytes = n_vec * (128 * 2 + L + engine.record_words(L, C) * 4)
    traffic2, traffic2_src = _ncu_traffic("cfg2", n_vec / 4_000_000)
    # e2e: the public build path from pinned host vectors (H2D inside the timed region),
    # reading back the last set offset
    import paper_2210_15748_b200 as dd
    Xh = X.cpu().pin_memory()
    cfg_e = dd.IndexConfig(d=128, C=C, L=L, seed=0, filter=dd.FilterConfig(enabled=False))
    ids_e = np.arange(len(sizes))
    dd.build_from_vectors(Xh.to(dev, non_blocking=True), sizes, ids_e, cfg_e, keep_codes=True,
                          hash_mode=mode)
    torch.cuda.synchronize()
    n_e2e = 5
    te = time.perf_counter()
    for _ in range(n_e2e):
        ie = dd.build_from_vectors(Xh.to(dev, non_blocking=True), sizes, ids_e, cfg_e,
                                   keep_codes=True, hash_mode=mode)
        tail = int(ie.set_off[-1].item())
    e2e_s = (time.perf_counter() - te) / n_e2e
    del ie, tail
    line = {
        "metric": "index-build vectors/sec (cfg2: 10M bf16 vectors, L=64 C=7, hash + CSR layout)",
        "value": n_vec / (ms * 1e-3), "unit": "vectors/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (cfg2-shaped, generated on GPU)",
        "config": {"workload": "cfg2", "vectors": n_vec, "sets": int(len(sizes)), "L": L, "C": C,
                   "hash_mode": "tcgen05 kind::f16, bf16 hi/lo planes (2 MMA chains)",
                   "l2": "inputs larger than L2 (2.56 GB)"},
        "roofline": {"bound": "tensor", "unit": "TFLOP/s", "kernel": "hash_tc_kernel<2,7,3>",
                     "kernel_ms": k_ms,
                     "achieved": alg_flops / (k_ms * 1e-3) / 1e12,
                     "peak": peaks["bf16_tflops"], "frac": alg_flops / (k_ms * 1e-3) / 1e12 / peaks["bf16_tflops"],
                     "mma_tflops_issued": mma_flops / (k_ms * 1e-3) / 1e12,
                     "mma_frac": mma_flops / (k_ms * 1e-3) / 1e12 / peaks["bf16_tflops"],
                     "hbm_gbs": hbm_bytes / (k_ms * 1e-3) / 1e9,
                     "hbm_frac": hbm_bytes / (k_ms * 1e-3) / 1e9 / peaks["hbm_gbs"],
                     "traffic": traffic2,
                     "traffic_detail": dict(traffic2_src or {}, algorithmic_bytes=hbm_bytes,
                                            ratio=None if traffic2 is None else traffic2 / hbm_bytes,
                                            note="X tiles are read by both 32-table groups' CTAs"),
                     "algorithmic": "2*d*L*C flops per vector; bytes 2d in + L codes + 4R records out",
                     "peak_source": "MEASURED_PEAKS.json bf16_tflops (burst), hbm_gbs"},
        "hash_bit_flips": {"sample_vectors": int(len(samp)), "bits": int(flips.size),
                           "flips": int(flips.sum()), "outside_band": int((flips & ~band).sum()),
                           "band_fraction": float(band.mean())},
        "e2e": {"value": n_vec / e2e_s, "unit": "vectors/s",
                "h2d_bytes_per_step": Xh.numel() * Xh.element_size(), "d2h_bytes_per_step": 8,
                "ms_per_step": e2e_s * 1e3,
                "path": "build_from_vectors (pinned host bf16 -> device, hash, layout)"},
        "clocks": clk, "gpu_launches": 4 * args.steps,
    }
    if not args.no_cpu_baseline:
        import bench_reference as BR

        r = BR.build_baseline(L=L, C=C)
        line["cpu_baseline"] = {"value": r["value"], "unit": "vectors/s", "cores": r["cores"],
                                "kind": r["kind"], "sample": r["sample"]}
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="cfg4: skip the cfg3 measurements in the line")
    ap.add_argument("--config", type=int, default=4, choices=[1, 2, 3, 4])
    ap.add_argument("--vectors", type=int, default=0, help="override cfg2 vector count")
    ap.add_argument("--sets", type=int, default=0, help="override N (cfg1/3/4)")
    ap.add_argument("--cpu-sets", type=int, default=20_000,
                    help="sets in the CPU reference sample (per step: 8 query sets x this)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--score-buffer", type=int, default=8 << 30)
    ap.add_argument("--latency-queries", type=int, default=1000)
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if args.config == 3:
        return run_cfg3(args)
    if args.config == 2:
        return run_cfg2(args)
    return run_scoring(args, args.config)


if __name__ == "__main__":
    sys.exit(main())
