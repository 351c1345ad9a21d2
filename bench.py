#!/usr/bin/env python
"""Quick ADC search benchmark on B200 (BASELINE.json metric: codes scanned/s
and QPS at N=1e9, with the scan kernel's roofline fraction).

Workload (default, N=1 GPU): BASELINE configs[4] — the metric's own
configuration, which fits one B200 (16 GB of codes + 8 GB of ids): IVF
K=65536 + OPQ, m=32 x 4-bit residual codes, N=10^9, Q=10^4 batched queries,
nprobe=64, R=100, init=1000. One step = one search_batch pass of all Q
queries (probe, residual + rotation + LUT, qmax, quantize, scan, exact
top-R). `--config cfg0..cfg3` selects the other BASELINE configs.

Multi-GPU (torchrun, one process per GPU, NCCL): configs[4] is range-sharded
(rank r holds its id range of every list, global list prefixes replicated;
strong scaling over the fixed N=10^9), configs[2] list-sharded, the
exhaustive configs range-sharded with a fixed N per GPU (weak scaling); the
per-rank top-R lists are merged exactly (all_gather over NCCL, (distance,
id) order). value = all codes scanned / max-over-ranks step time.

Beside the device number the line carries: `e2e` (host queries in, host
results out, through the public API), `roofline` (the scan kernel vs the
measured integer-issue or int8-MMA peak, plus the HBM view), `cpu_baseline`
(the reference's compiled qadc_scan_u8 driven by the restated adc.search
orchestration on the host cores, on a query sample of the same index), and
`parity` (the GPU's results and tables against the reference's semantics
on that sample: ids / distance bits, fp32 LUT bits, uint8 flips, qmax).

`--impl reference` times the reference's CPU path alone (rank 0): the same
workload built with plain torch (no product library in that process), the
same query sample scheme, all host threads.
"""

from __future__ import annotations

import os

# the stock reference's numpy runs single-threaded per worker process
# (one process per core, OPENBLAS_NUM_THREADS=1)
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

import argparse
import json
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRICS = {
    "cfg0": "Quick ADC codes scanned/s (whole job) at configs[0]: exhaustive, m=16x4-bit, N=1e6, Q=100, R=100",
    "cfg1": "Quick ADC codes scanned/s (whole job) at configs[1]: exhaustive, m=32x4-bit, N=1e7/GPU, Q=1000, R=100",
    "cfg2": "Quick ADC codes scanned/s (whole job) at configs[2]: IVF K=4096 + OPQ, m=32x4-bit, Q=1e4, R=100",
    "cfg3": "Quick ADC codes scanned/s (whole job) at configs[3]: exhaustive, d=960, m=32x4-bit, N=1e6, Q=1000, R=100",
    "cfg4": "Quick ADC codes scanned/s (whole job) at configs[4]: IVF K=65536 + OPQ, m=32x4-bit, N=1e9 range-sharded, Q=1e4, nprobe=64, R=100",
}
DEFAULT_CONFIG = "cfg4"
METRIC = METRICS[DEFAULT_CONFIG]
UNIT = "codes/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--config", default=DEFAULT_CONFIG,
                   choices=["cfg0", "cfg1", "cfg2", "cfg3", "cfg4"])
    p.add_argument("--nprobe", type=int, default=None, help="IVF configs: probed cells (ma)")
    p.add_argument("--n", type=int, default=None,
                   help="codes per GPU (exhaustive) / in total (IVF); default: the config's N")
    p.add_argument("--queries", type=int, default=None)
    p.add_argument("--cpu-seconds", type=float, default=12.0,
                   help="target CPU work of the bounded reference sample")
    p.add_argument("--parity-queries", type=int, default=200,
                   help="IVF configs: queries of the native-mode parity accounting")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--replicate-tables", action="store_true",
                   help="N>1: every rank prepares the whole batch (default: the Index + Tables "
                        "phases are split by query and all-gathered, dist.sharded_prepare)")
    p.add_argument("--recall", type=int, default=0,
                   help="report R@1/10/100 on this many queries (exact GPU ground truth)")
    return p.parse_args()


# ---------------------------------------------------------------- clocks

class ClockSampler:
    """SM clock and throttle reasons sampled (NVML, every 100 ms) during the
    timed region; falls back to nvidia-smi if NVML is unavailable."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap"}

    def __init__(self, index: int):
        self.index = index
        self.sm, self.mx, self.reasons = [], [], set()
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            while not self._stop.is_set():
                self.sm.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                self.mx.append(mx)
                r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.reasons.update(v for k, v in self.REASONS.items() if r & k)
                self._stop.wait(0.1)
        except Exception:
            while not self._stop.is_set():
                try:
                    out = subprocess.run(
                        ["nvidia-smi", f"--id={self.index}",
                         "--query-gpu=clocks.sm,clocks.max.sm", "--format=csv,noheader,nounits"],
                        capture_output=True, text=True, timeout=5).stdout.split(",")
                    self.sm.append(float(out[0]))
                    self.mx.append(float(out[1]))
                except Exception:
                    pass
                self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        time.sleep(0.05)
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        return {"sm_mhz": statistics.median(self.sm) if self.sm else None,
                "sm_max_mhz": max(self.mx) if self.mx else None,
                "reasons": sorted(self.reasons), "samples": len(self.sm)}


# ---------------------------------------------------------------- helpers

def measured_peaks():
    f = ROOT / "MEASURED_PEAKS.json"
    if f.exists():
        try:
            return json.loads(f.read_text())
        except Exception:
            pass
    return {"hbm_gbs": 6650.0, "fallback": True}


def ncu_traffic(config):
    """Per-launch DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum)
    of this config's scan kernel from its own committed `ncu --set full`
    summary (profiles/scan_ncu_<config>.json), or None."""
    f = ROOT / "profiles" / f"scan_ncu_{config}.json"
    if f.exists():
        try:
            return json.loads(f.read_text()).get("dram_bytes_per_launch")
        except Exception:
            return None
    return None


def host_info():
    """CPU model, thread count and the numpy / OpenBLAS build the CPU
    baseline ran with (the reference's arithmetic depends on them)."""
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    blas = None
    try:
        import ctypes
        import glob
        for f in glob.glob(os.path.join(os.path.dirname(np.__file__), "..", "numpy.libs",
                                        "libscipy_openblas*.so")):
            L = ctypes.CDLL(f)
            fn = getattr(L, "scipy_openblas_get_config64_", None) or getattr(
                L, "scipy_openblas_get_config", None)
            if fn is not None:
                fn.restype = ctypes.c_char_p
                blas = fn().decode()
    except Exception:
        pass
    return {"cpu_model": model, "threads": os.cpu_count(), "numpy": np.__version__,
            "openblas": blas}


def _product_lib_mapped() -> bool:
    """Whether libqadc_b200.so is mapped into this process (the reference
    arm must never load it)."""
    try:
        return "libqadc_b200" in open("/proc/self/maps").read()
    except OSError:
        return False


def config_of(cfg, ivf_cfg, n, nq, ma, world):
    """The workload's config dict, identical in both arms."""
    c = {"workload": cfg.name, "m": cfg.m, "d": cfg.mix.d, "Q": nq, "R": cfg.R,
         "init": cfg.init, "nprobe": ma}
    if ivf_cfg is not None:
        c.update({"K": ivf_cfg.K, "N_total": n,
                  "sharding": ivf_cfg.sharding + (" (strong)" if world > 1 else "")})
    else:
        c.update({"N_per_gpu": n, "N_total": n * world,
                  "sharding": "range (weak)" if world > 1 else "none"})
    return c


def host_lists(rows, ids, row_off, lists):
    """Oracle-layout (blocks, blk_off, ids, count) of the given lists of a
    row-ordered device index (every other list empty): the oracle's result
    and work for queries probing only these lists equal those of the full
    index. Returns (flat, list sizes of the full index)."""
    import torch

    from paper_1704_07355_b200.qadc import transpose_list
    from paper_1704_07355_b200.shard import _ranges

    K = row_off.shape[0] - 1
    want = np.zeros(K, bool)
    want[np.unique(np.asarray(lists))] = True
    off = row_off.cpu().numpy()
    sizes = np.diff(off)
    sel = torch.from_numpy(np.nonzero(want)[0]).to(row_off.device)
    idx = _ranges(row_off[:-1][sel], row_off[1:][sel] - row_off[:-1][sel])
    r_h, i_h = rows[idx].cpu().numpy(), ids[idx].cpu().numpy()
    blocks, bids, boff, count = [], [], [0], []
    o = 0
    for L in range(K):
        k = int(sizes[L]) if want[L] else 0
        if k:
            tl = transpose_list(r_h[o:o + k], i_h[o:o + k])
            blocks.append(tl.blocks.reshape(-1))
            bids.append(tl.ids)
            boff.append(boff[-1] + tl.blocks.shape[0])
            o += k
        else:
            boff.append(boff[-1])
        count.append(k)
    flat = (np.concatenate(blocks) if blocks else np.zeros(0, np.uint8), np.asarray(boff, np.int64),
            np.concatenate(bids) if bids else np.zeros(0, np.int64), np.asarray(count, np.int64))
    return flat, sizes


# ---------------------------------------------------------------- stock reference

STOCK = ROOT / "baseline" / "_ref"  # pip install --target of /root/reference/pkg (git-ignored)


def stock_reference():
    """The UNMODIFIED reference package (`qadc`, installed by
    `pip install --no-index --no-build-isolation --no-deps --target
    baseline/_ref /root/reference/pkg`), or None if it is not installed."""
    if not (STOCK / "qadc").exists():
        return None
    if str(STOCK) not in sys.path:
        sys.path.insert(0, str(STOCK))
    try:
        import qadc
        from qadc import kernels
        if not kernels.have_extension():
            return None
        return qadc
    except Exception:
        return None


def stock_index(coarse, m, d, rows, ids, row_off, lists):
    """A reference IvfIndex (transposed16 layout) holding the given lists of
    a row-ordered device index (every other list empty); flat when coarse
    is None."""
    from qadc import ivf, kmeans
    from qadc import qadc as rq

    off = row_off.cpu().numpy()
    K = off.shape[0] - 1
    want = np.zeros(K, bool)
    want[np.unique(np.asarray(lists))] = True
    empty = rq.transpose_list(np.zeros((0, m // 2), np.uint8), np.zeros(0, np.int64))
    out = []
    for L in range(K):
        a, b = int(off[L]), int(off[L + 1])
        if want[L] and b > a:
            out.append(rq.transpose_list(rows[a:b].cpu().numpy(), ids[a:b].cpu().numpy()))
        else:
            out.append(empty)
    cb = None if coarse is None else kmeans.Codebook(np.ascontiguousarray(coarse, np.float32))
    return ivf.IvfIndex(d=d, m=m, b=4, coarse=cb, lists=out, layout=ivf.LAYOUT_TRANSPOSED)


_STOCK = {}


def _stock_worker(task):
    from qadc import adc
    idx, pq, R, ma, init = (_STOCK[k] for k in ("index", "pq", "R", "ma", "init"))
    lo, qs = task
    out = []
    for q in qs:
        r = adc.search(idx, pq, q, R=R, ma=ma, method="qadc", init=init, variant="simd256")
        out.append((r.ids, r.distances))
    return lo, out


def stock_pool(ref_index, codebooks, rotation, R, ma, init, nq):
    """A fork pool of one worker process per core (at most nq) sharing the
    reference index copy-on-write; returns (pool, pq, procs)."""
    import multiprocessing as mp

    from qadc import pq as rpq
    pq = rpq.ProductQuantizer(m=codebooks.shape[0], b=4, codebooks=codebooks, rotation=rotation)
    procs = max(1, min(os.cpu_count() or 1, nq))
    _STOCK.update(index=ref_index, pq=pq, R=R, ma=ma, init=init)
    return mp.get_context("fork").Pool(procs), pq, procs


def stock_all_cores(pool, procs, qs, R):
    """One pass of the stock adc.search over qs on the worker pool (disjoint
    contiguous slices); returns (wall seconds, ids, dists padded to R)."""
    per = -(-qs.shape[0] // procs)
    tasks = [(i, qs[i:i + per]) for i in range(0, qs.shape[0], per)]
    t0 = time.perf_counter()
    parts = pool.map(_stock_worker, tasks)
    wall = time.perf_counter() - t0
    ri = np.full((qs.shape[0], R), -1, np.int64)
    rd = np.full((qs.shape[0], R), np.inf, np.float32)
    for lo, out in parts:
        for j, (i_, d_) in enumerate(out):
            ri[lo + j, : i_.shape[0]] = i_
            rd[lo + j, : d_.shape[0]] = d_
    return wall, ri, rd


def stock_single_core(ref_index, pq, qs, R, ma, init, codes_per_query):
    """The stock adc.search sequentially on one core with the reference's
    own Index / Tables / Scan phase times (bench.py:176-192)."""
    from qadc import adc
    ph = np.zeros(3)
    t0 = time.perf_counter()
    for q in qs:
        r = adc.search(ref_index, pq, q, R=R, ma=ma, method="qadc", init=init, variant="simd256")
        ph += (r.timings.index_ms, r.timings.tables_ms, r.timings.scan_ms)
    wall = time.perf_counter() - t0
    n = qs.shape[0]
    return {"queries": n, "qps": n / wall,
            "codes_per_s": float(np.sum(codes_per_query[:n])) / wall,
            "index_ms": round(ph[0] / n, 3), "tables_ms": round(ph[1] / n, 3),
            "scan_ms": round(ph[2] / n, 3), "total_ms": round(wall * 1e3 / n, 3)}


def stock_baseline(ref_index, codebooks, rotation, qs_single, qs_all, R, ma, init,
                   codes_per_query, seconds):
    """SURVEY 8d CPU baseline with the stock reference: single-core phases
    and all-core throughput (one process per core, passes repeated for
    about `seconds`). Returns (cpu_baseline dict, all-core results)."""
    pool, pq, procs = stock_pool(ref_index, codebooks, rotation, R, ma, init, qs_all.shape[0])
    try:
        single = stock_single_core(ref_index, pq, qs_single, R, ma, init, codes_per_query)
        walls, res = [], None
        t_end = time.perf_counter() + seconds
        while True:
            w, ri, rd = stock_all_cores(pool, procs, qs_all, R)
            walls.append(w)
            res = (ri, rd)
            if time.perf_counter() >= t_end:
                break
    finally:
        pool.close()
        pool.join()
    wall = statistics.median(walls)
    codes = float(np.sum(codes_per_query[: qs_all.shape[0]]))
    return {"value": codes / wall, "unit": UNIT, "cores": procs, "kind": "reference",
            "qps": qs_all.shape[0] / wall, "passes": len(walls),
            "single_core": single}, res


POOL = 512  # IVF configs: queries of the CPU sample (both arms) and its list extraction


def _time_cpu(fn, seconds):
    """Run fn() (one pass over the sample) until `seconds` of wall time
    accumulated (at least once); returns (last result, wall per pass)."""
    walls, out = [], None
    t_end = time.perf_counter() + seconds
    while True:
        t0 = time.perf_counter()
        out = fn()
        walls.append(time.perf_counter() - t0)
        if time.perf_counter() >= t_end:
            break
    return out, statistics.median(walls), len(walls)


def cpu_reference_run(cb, flat, n, qs, R, init, seconds, nthreads=None):
    """Exhaustive CPU baseline: the reference's compiled qadc_scan_u8
    (oracle/_ref) driven by the restated adc.search orchestration (oracle/)
    on all host threads, over the full index, on the largest query prefix
    that fits `seconds` of CPU work."""
    from oracle import oracle as orc

    use_ref = orc.ref_lib() is not None
    nthreads = nthreads or os.cpu_count() or 1
    probe = qs[: max(1, min(nthreads, qs.shape[0]))]
    t0 = time.perf_counter()
    orc.search_batch(probe, cb, None, None, 1, flat, R, init, use_ref_scan=use_ref,
                     nthreads=nthreads)
    per_q = (time.perf_counter() - t0) / probe.shape[0]
    nq = int(max(probe.shape[0], min(qs.shape[0], seconds / max(per_q, 1e-6))))
    sample = qs[:nq]
    t0 = time.perf_counter()
    oi, od, on, _ = orc.search_batch(sample, cb, None, None, 1, flat, R, init,
                                     use_ref_scan=use_ref, nthreads=nthreads)
    wall = time.perf_counter() - t0
    return {"value": nq * n / wall, "unit": UNIT, "cores": nthreads,
            "kind": "reference" if use_ref else "port",
            "sample": f"{nq} of {qs.shape[0]} queries over the full N={n} index",
            "seconds": round(wall, 2)}, (oi, od, on), nq


def cpu_reference_run_ivf(pq, coarse, flat, sizes, pool, cells, R, init, ma, seconds, nq_total,
                          nthreads=None):
    """IVF CPU baseline: the restated adc.search orchestration (probe,
    residual, OPQ rotation in OpenBLAS sgemv order, tables, qmax,
    quantization; oracle/) with the reference's own compiled qadc_scan_u8
    (oracle/_ref) as the block scan, all host threads, over the POOL
    queries (their probed lists extracted from the full index), repeated
    for about `seconds`. codes/s counts (query, probed list) codes."""
    from oracle import oracle as orc

    use_ref = orc.ref_lib() is not None
    nthreads = nthreads or os.cpu_count() or 1
    codes = int(sizes[np.asarray(cells)].sum())

    def one():
        return orc.search_batch(pool, pq.codebooks, pq.rotation, coarse, ma, flat, R, init,
                                use_ref_scan=use_ref, nthreads=nthreads)
    (oi, od, on, _), wall, reps = _time_cpu(one, seconds)
    return {"value": codes / wall, "unit": UNIT, "cores": nthreads,
            "kind": "reference" if use_ref else "port",
            "sample": f"{pool.shape[0]} of {nq_total} queries, nprobe={ma}, over the lists they "
                      f"probe of the full index ({reps} passes, median)",
            "seconds": round(wall * reps, 2)}, (oi, od, on)


def ivf_parity(index, pq, coarse, flat, pool, R, init, ma, gpu_i, gpu_d, cpu_res, nparity):
    """Native-mode parity of the GPU against the reference on the pool:
    (1) results vs the timed CPU reference run; (2) on the first
    `nparity` queries, the GPU's tables vs the reference's Index + Tables
    phases re-run with THIS host's numpy rotation (adc.py:108-111; counts
    of fp32 LUT bit mismatches, uint8 flips, qmax mismatches, max LUT
    relative error) and the results vs the oracle fed those tables; (3) a
    reference-LUT-injected GPU run on the same queries (must be exact)."""
    import torch

    from oracle import oracle as orc
    from oracle import parity

    oi, od, _ = cpu_res
    out = {"vs_cpu_reference": parity.compare_results(gpu_i[: oi.shape[0]], gpu_d[: oi.shape[0]],
                                                      oi, od)}
    k = min(nparity, pool.shape[0])
    qk = pool[:k]
    t = {a: b.cpu().numpy() for a, b in index.tables(torch.from_numpy(qk).cuda(), R, ma=ma,
                                                     init=init).items()}
    ref = parity.reference_tables(qk, pq.codebooks, pq.rotation, coarse, ma, flat, R, init)
    acc = parity.account(t, ref)
    ri, rd, _, _ = orc.search_batch(qk, pq.codebooks, pq.rotation, coarse, ma, flat, R, init,
                                    lut_in=ref["lut"], cells_in=ref["cells"],
                                    nthreads=os.cpu_count())
    out["native_tables_vs_host_blas"] = {a: b for a, b in acc.items() if not a.startswith("_")}
    out["native_results_vs_host_blas"] = parity.compare_results(gpu_i[:k], gpu_d[:k], ri, rd,
                                                                acc["_diverged"])
    inj = index.search(torch.from_numpy(qk).cuda(), R, ma=ma, init=init,
                       lut=torch.from_numpy(ref["lut"]).cuda(),
                       cells=torch.from_numpy(ref["cells"]).cuda())
    out["lut_injected"] = parity.compare_results(inj.ids.cpu().numpy(),
                                                 inj.distances.cpu().numpy(), ri, rd)
    return out


def measure_recall(cfg, pq, n, qs, ids, codes=None):
    """R@{1,10,100} (reference bench.py:110-122) against exact float64
    nearest neighbours of the same GPU-drawn base (regenerated chunk by
    chunk with the build's seeds, recall.ground_truth = synth.py:45-70's
    definition). For a flat index (`codes` given) the float-table ADC
    top-100 of the same codes is measured too, so the quantized-table
    recall loss (the paper's QADC vs ADC figure) sits beside it."""
    import torch

    from paper_1704_07355_b200.adc import compute_tables
    from paper_1704_07355_b200.recall import ground_truth, recall_at
    from paper_1704_07355_b200.workload import base_chunks

    gt = ground_truth(base_chunks(cfg, n), qs, depth=1)[:, 0]
    out = {f"R@{r}": recall_at(ids, gt, r) for r in (1, 10, 100)}
    if codes is not None:
        T = torch.from_numpy(np.stack([compute_tables(pq, q).tables for q in qs])).cuda()
        best_d, best_i = None, None
        for c0 in range(0, n, 1 << 21):
            c = codes[c0:c0 + (1 << 21)]
            sub = torch.stack([c & 15, c >> 4], 2).reshape(c.shape[0], -1).long()
            acc = torch.zeros((T.shape[0], c.shape[0]), device="cuda")
            for j in range(pq.m):
                acc += T[:, j, :][:, sub[:, j]]
            dd, ii = torch.topk(acc, min(100, c.shape[0]), dim=1, largest=False)
            ii = ii + c0
            if best_d is not None:
                dd, ii = torch.cat([best_d, dd], 1), torch.cat([best_i, ii], 1)
                o = torch.topk(dd, 100, dim=1, largest=False).indices
                dd, ii = torch.gather(dd, 1, o), torch.gather(ii, 1, o)
            best_d, best_i = dd, ii
        o = torch.argsort(best_d, dim=1, stable=True)
        fi = torch.gather(best_i, 1, o).cpu().numpy()
        out["adc_float"] = {f"R@{r}": recall_at(fi, gt, r) for r in (1, 10, 100)}
    return out | {"queries": int(qs.shape[0])}


def run_b200(args):
    import torch
    import torch.distributed as dist

    from paper_1704_07355_b200 import _native
    from paper_1704_07355_b200.dist import merge_topr, sharded_prepare
    from paper_1704_07355_b200.workload import (BUILD_TIMES, CONFIGS, IVF_CONFIGS,
                                                build_ivf_index, build_shard_index,
                                                build_sharded_ivf_index, load_ivf_model, load_pq,
                                                queries)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # developer check of the multi-rank logic on a one-GPU box (not a
    # measurement): QADC_BENCH_BACKEND=gloo QADC_BENCH_ONE_DEVICE=1
    if os.environ.get("QADC_BENCH_ONE_DEVICE") == "1":
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        backend = os.environ.get("QADC_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    _native.require_device()
    ivf_cfg = IVF_CONFIGS.get(args.config)
    cfg = ivf_cfg or CONFIGS[args.config]
    n = args.n or cfg.n
    nq = args.queries or cfg.q
    R, init = cfg.R, cfg.init
    ma = 1
    t_build = time.perf_counter()
    if ivf_cfg is not None:
        ma = args.nprobe or ivf_cfg.nprobe
        pq, coarse = load_ivf_model(ivf_cfg)
        if world > 1:
            index, rows, row_ids, row_off = build_sharded_ivf_index(
                ivf_cfg, pq, coarse, n, rank, world, prefix=max(init, R))
        else:
            index, sizes, rows, row_ids, row_off = build_ivf_index(ivf_cfg, pq, coarse, n)
    else:
        pq = load_pq(cfg)
        index, codes = build_shard_index(cfg, pq, n, rank, world, prefix=max(init, R))
    torch.cuda.synchronize()
    t_build = time.perf_counter() - t_build
    qs = queries(cfg, nq)
    q_dev = torch.from_numpy(qs).cuda()
    q_pin = torch.from_numpy(qs).pin_memory()
    torch.cuda.synchronize()

    shard_tables = world > 1 and not args.replicate_tables

    def search(q):
        if shard_tables:  # query-sharded Index + Tables phases, then the local scan
            return index.scan(sharded_prepare(index, q, R, ma, init), R, ma=ma, init=init)
        return index.search(q, R, ma=ma, init=init, with_fsat=(rank == 0))

    def step_device():
        res = search(q_dev)
        gi, gd, _ = merge_topr(res.ids, res.distances, R)
        return (gi, gd), res

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        step_device()
    torch.cuda.synchronize()

    # ---- device-resident timed region ----
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st = {k: 0 for k in ("scan_us", "launches", "codes", "candidates", "reruns", "probe_us",
                         "tables_us", "work_us", "select_us")}
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        torch.cuda.nvtx.range_push("qadc_timed_region")  # ncu --nvtx --nvtx-include "qadc_timed_region/"
        e0.record(stream)
        for _ in range(args.steps):
            (gi, gd), res = step_device()
            for k in st:
                st[k] += res.stats[k]
        e1.record(stream)
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_pop()
    barrier()
    ms_dev = max_over_ranks(e0.elapsed_time(e1) / args.steps)

    # ---- end-to-end through the public API with host buffers ----
    out_i_pin = torch.empty((nq, R), dtype=torch.int64).pin_memory()
    out_d_pin = torch.empty((nq, R), dtype=torch.float32).pin_memory()

    def step_e2e():
        qd = q_pin.to("cuda", non_blocking=True)
        res = search(qd)
        gi, gd, _ = merge_topr(res.ids, res.distances, R)
        out_i_pin.copy_(gi, non_blocking=True)
        out_d_pin.copy_(gd, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return out_i_pin, out_d_pin

    for _ in range(args.warmup):
        step_e2e()
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    e2.record(stream)
    for _ in range(args.steps):
        out_i, out_d = step_e2e()
    e3.record(stream)
    torch.cuda.synchronize()
    barrier()
    ms_e2e = max_over_ranks(e2.elapsed_time(e3) / args.steps)

    # codes scanned per step = sum over (query, probed list) of len(list),
    # counted by the library on each rank's own codes, summed over ranks
    per_rank_codes = st["codes"] / args.steps
    total_codes = per_rank_codes
    if world > 1:
        t = torch.tensor([per_rank_codes], dtype=torch.float64, device="cuda")
        dist.all_reduce(t)
        total_codes = float(t.item())
    value = total_codes / (ms_dev * 1e-3)
    e2e_value = total_codes / (ms_e2e * 1e-3)

    # ---- roofline of the dominant kernel (the scan) ----
    peak = np.zeros(2, np.float64)
    lib = _native.load_library()
    _native.check(lib.qadc_b200_int_peak(peak.ctypes.data_as(_native._f64p)), "int_peak")
    scan_s = st["scan_us"] / args.steps * 1e-6
    pairs = per_rank_codes  # (query, code) pairs per launch, this rank
    lookups = pairs * pq.m
    pk = measured_peaks()
    # codes of every DISTINCT list touched once per batch
    hbm_bytes = index.ncodes * pq.m / 2
    int_view = {"achieved_G_lookups": round(lookups / scan_s / 1e9, 2),
                "peak_G_lane_instr": round(peak[0] / 1e9, 2),
                "frac": round(lookups / scan_s / peak[0], 4),
                "alu_pipe_peak_G": round(peak[1] / 1e9, 2)}
    if res.stats.get("scan_tc") == 2:
        # k_scan_tcw (IVF lists probed by a few queries each): every list is
        # scanned ceil(pairs / tq) times (tq = 32 queries per pass); a pass
        # expands each code of the
        # list into its one-hot A row (4 m PRMT per code on the ALU pipe) and
        # runs m / 2 MMAs of N = 16 or 32 per 128-code tile. Three ceilings:
        # executed int8 MMA ops vs the measured tensor peak (the contract's
        # "tensor" bound), the expansion's PRMTs vs the measured ALU-pipe
        # rate, and the code bytes vs HBM; plus north_star's integer-issue
        # view (lookups / R_int), which this kernel may exceed because the
        # lookups run on the tensor pipe.
        mma = np.zeros(1, np.float64)
        _native.check(lib.qadc_b200_mma_peak(mma.ctypes.data_as(_native._f64p)), "mma_peak")
        cells_l = index.tables(q_dev, R, ma=ma, init=init)["cells"].cpu().numpy().ravel()
        sizes_l = np.diff(row_off.cpu().numpy())
        pl = np.bincount(cells_l, minlength=sizes_l.size)
        tiles = 2 * ((sizes_l + 255) // 256)
        tq = int(res.stats.get("scan_tile_q") or 32)  # queries per pass over a list
        full, rem = pl // tq, pl % tq
        ncols = tq * full + ((rem + 15) // 16) * 16  # MMA N of the last pass: rounded to 16
        passes = full + (rem > 0)
        ops_exec = float((tiles * ncols).sum()) * 128 * 16 * pq.m * 2
        ops_useful = pairs * 16 * pq.m * 2
        code_passes = float((tiles * passes).sum()) * 128
        prmt = code_passes * 4 * pq.m
        cm_bytes = code_passes * pq.m / 2
        hbm_peak = pk.get("hbm_gbs", 6650.0) * 1e9
        t_tensor, t_alu, t_hbm = ops_exec / mma[0], prmt / peak[1], cm_bytes / hbm_peak
        roof = {"bound": "tensor", "achieved": round(ops_exec / scan_s / 1e12, 2),
                "peak": round(mma[0] / 1e12, 2),
                "unit": "TOP/s int8 (executed one-hot MMA ops: 128 codes x N (queries of the pass, "
                        "rounded to 16) x 16 m per tile and pass) vs measured tcgen05.mma.kind::i8 peak "
                        "(qadc_b200_mma_peak)",
                "frac": round(t_tensor / scan_s, 4),
                "useful_ops_frac": round(ops_useful / scan_s / mma[0], 4),
                "alu_expansion_view": {"prmt_lane_instr": int(prmt),
                                       "alu_pipe_peak_G": int_view["alu_pipe_peak_G"],
                                       "frac": round(t_alu / scan_s, 4)},
                "roof_ms": {"tensor": round(t_tensor * 1e3, 2), "alu_expansion": round(t_alu * 1e3, 2),
                            "hbm_code_major": round(t_hbm * 1e3, 2),
                            "north_star_int_issue": round(lookups / peak[0] * 1e3, 2)},
                "frac_of_slowest_ceiling": round(max(t_tensor, t_alu, t_hbm) / scan_s, 4),
                "list_passes": {"queries_per_pass": tq, "code_passes": int(code_passes),
                                "mean_passes_per_scanned_code":
                                round(code_passes / max(1.0, float((tiles * (pl > 0)).sum()) * 128), 3)},
                "int_issue_view": int_view}
        hbm_bytes = cm_bytes
    elif res.stats.get("scan_tc"):
        # int8 tcgen05 one-hot GEMM: 16 m MACs (2 ops each) per (query, code)
        # pair; achieved = useful ops / launch time vs the measured int8 rate
        mma = np.zeros(1, np.float64)
        _native.check(lib.qadc_b200_mma_peak(mma.ctypes.data_as(_native._f64p)), "mma_peak")
        ops = pairs * 16 * pq.m * 2
        roof = {"bound": "tensor", "achieved": round(ops / scan_s / 1e12, 2),
                "peak": round(mma[0] / 1e12, 2),
                "unit": "TOP/s int8 (one-hot MMA ops of the scanned pairs) vs measured "
                        "tcgen05.mma.kind::i8 peak (qadc_b200_mma_peak)",
                "frac": round(ops / scan_s / mma[0], 4),
                "int_issue_view": int_view}
    else:
        roof = {"bound": "int", "achieved": int_view["achieved_G_lookups"],
                "peak": int_view["peak_G_lane_instr"],
                "unit": "G lookup-adds/s (m per scanned (query, code) pair) vs measured G int "
                        "lane-instr/s (PRMT+IMAD dual-pipe microbench, qadc_b200_int_peak)",
                "frac": int_view["frac"], "alu_pipe_peak_G": int_view["alu_pipe_peak_G"]}
    roof.update({
        "kernel": {0: "k_scan (PRMT)", 1: "k_scan_tc2 / k_scan_tc", 2: "k_scan_tcw"}[
            int(res.stats.get("scan_tc", 0))],
        "traffic": ncu_traffic(args.config),
        "scan_kernel_ms": round(scan_s * 1e3, 3),
        "algorithmic_units_per_launch": {"pairs": int(pairs), "lookups": int(lookups)},
        "hbm": {"bytes_alg_per_launch": int(hbm_bytes),
                "achieved_gbs": round(hbm_bytes / scan_s / 1e9, 1),
                "peak_gbs": pk.get("hbm_gbs"),
                "frac": round(hbm_bytes / scan_s / 1e9 / pk.get("hbm_gbs", 6650.0), 4)},
        "scan_share_of_step": round(scan_s * 1e3 / ms_dev, 3),
    })

    out = None
    if rank == 0:
        ph = {k: round(st[k] / args.steps / 1e3, 3) for k in ("probe_us", "tables_us", "work_us",
                                                             "scan_us", "select_us")}
        out = {
            "metric": METRICS[args.config], "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_dev,
            "higher_is_better": True, "scaling": "weak" if ivf_cfg is None else "strong",
            "vs_baseline": None, "dtype": "u8",
            "data": "synthetic (BASELINE mixture generator drawn on the GPU, seeded; " + (
                "PQ codebooks trained by the reference's train_pq)" if ivf_cfg is None else
                f"coarse K={ivf_cfg.K} by GPU Lloyd (tools/train_coarse.py), seeded orthogonal "
                "OPQ rotation, residual PQ codebooks by the reference's train_pq; see DESIGN.md)"),
            "config": config_of(cfg, ivf_cfg, n, nq, ma, world),
            "tables_phase": ("query-sharded + all_gather" if shard_tables else
                             ("replicated on every rank" if world > 1 else "local")),
            "qps": nq / (ms_dev * 1e-3),
            "e2e": {"value": e2e_value, "unit": UNIT, "qps": nq / (ms_e2e * 1e-3),
                    "ms_per_step": ms_e2e, "h2d_bytes_per_step": int(nq * pq.d * 4),
                    "d2h_bytes_per_step": int(nq * R * 12)},
            "roofline": roof,
            "phases_ms": {"probe": ph["probe_us"], "tables": ph["tables_us"],
                          "work_list": ph["work_us"], "scan": ph["scan_us"],
                          "select": ph["select_us"]},
            "clocks": clk.summary(),
            "gpu_launches": int(st["launches"]),
            "candidates_per_query": st["candidates"] / max(1, args.steps * nq),
            "reruns": st["reruns"],
            "workload_notes": {
                "codes_scanned_per_step": int(total_codes),
                "index_build_s": round(t_build, 1),
                "index_build_phases_s": {k: round(v, 1) for k, v in BUILD_TIMES.items()},
                "l2": "inputs larger than L2 (codes %.0f MB > 126 MB)" % (hbm_bytes / 1e6)
                if hbm_bytes > 126e6 else
                "index %.0f MB fits L2: steady-state (L2-warm) throughput" % (hbm_bytes / 1e6)},
        }
        if world == 1 and not args.no_cpu_baseline:
            out["cpu_host"] = host_info()
            from oracle import parity
            gi_np, gd_np = out_i.numpy(), out_d.numpy()
            if ivf_cfg is not None:
                pool = qs[: min(POOL, nq)]
                t = index.tables(torch.from_numpy(pool).cuda(), R, ma=ma, init=init)
                cells = t["cells"].cpu().numpy()
                flat, sizes = host_lists(rows, row_ids, row_off, cells)
                cb_res, cpu_res = cpu_reference_run_ivf(pq, coarse, flat, sizes, pool, cells, R,
                                                        init, ma, args.cpu_seconds, nq)
                out["parity"] = ivf_parity(index, pq, coarse, flat, pool, R, init, ma, gi_np,
                                           gd_np, cpu_res, args.parity_queries)
                codes_pq = sizes[cells].sum(1)
                if stock_reference() is not None:
                    ref_index = stock_index(coarse, pq.m, pq.d, rows, row_ids, row_off, cells)
                    n1, na = min(16, pool.shape[0]), min(256, pool.shape[0])
                    st_res, (si, sd) = stock_baseline(ref_index, pq.codebooks, pq.rotation,
                                                      pool[:n1], pool[:na], R, ma, init, codes_pq,
                                                      args.cpu_seconds / 2)
                    st_res["sample"] = (f"{na} of {nq} queries (single core: {n1}), nprobe={ma}, "
                                        "over the lists they probe of the full index: the stock "
                                        "reference package (baseline/_ref) adc.search(method="
                                        "'qadc', variant='simd256'), one process per core")
                    st_res["restated_kernels"] = cb_res
                    out["cpu_baseline"] = st_res
                    out["parity"]["vs_stock_reference"] = parity.compare_results(
                        gi_np[:na], gd_np[:na], si, sd)
                else:
                    out["cpu_baseline"] = cb_res
            else:
                from paper_1704_07355_b200.qadc import transpose_list
                tl = transpose_list(codes.cpu().numpy(), np.arange(n, dtype=np.int64))
                flat = (tl.blocks.reshape(-1), np.array([0, tl.blocks.shape[0]], np.int64),
                        tl.ids, np.array([n], np.int64))
                cb_res, (oi, od, on), k = cpu_reference_run(pq.codebooks, flat, n, qs, R, init,
                                                            args.cpu_seconds)
                out["parity"] = {"vs_cpu_reference": parity.compare_results(
                    gi_np[:k], gd_np[:k], oi, od)}
                if stock_reference() is not None:
                    ids_d = torch.arange(n, dtype=torch.int64)
                    ref_index = stock_index(None, pq.m, pq.d, codes, ids_d,
                                            torch.tensor([0, n]), [0])
                    n1, na = min(4, nq), min(64, nq)
                    st_res, (si, sd) = stock_baseline(ref_index, pq.codebooks, None, qs[:n1],
                                                      qs[:na], R, 1, init, np.full(nq, n),
                                                      args.cpu_seconds / 2)
                    st_res["sample"] = (f"{na} of {nq} queries (single core: {n1}) over the full "
                                        f"N={n} index: the stock reference package "
                                        "(baseline/_ref) adc.search(method='qadc', "
                                        "variant='simd256'), one process per core")
                    st_res["restated_kernels"] = cb_res
                    out["cpu_baseline"] = st_res
                    out["parity"]["vs_stock_reference"] = parity.compare_results(
                        gi_np[:na], gd_np[:na], si, sd)
                else:
                    out["cpu_baseline"] = cb_res
    if out is not None and args.recall and world == 1:
        out["recall"] = measure_recall(cfg, pq, n, qs[: args.recall], out_i.numpy()[: args.recall],
                                       codes=None if ivf_cfg is not None else codes)
    if world > 1:
        dist.destroy_process_group()
    return out


def run_reference(args):
    """CPU reference arm, rank 0 only: the stock reference package
    (baseline/_ref: `pip install --no-deps --target` of /root/reference/pkg)
    running its own adc.search(method="qadc", variant="simd256"), one
    process per host core, on a bounded query sample per step (the
    restated orchestration with the reference's compiled scan kernels,
    oracle/ + oracle/_ref, if the stock package is absent). The index is
    built in plain torch on the GPU (workload.ivf_rows_torch /
    encode_torch): no product kernel runs, and libqadc_b200.so is never
    loaded, in this process."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return None
    import torch

    from paper_1704_07355_b200.workload import (CONFIGS, IVF_CONFIGS, encode_torch,
                                                ivf_rows_torch, load_ivf_model, load_pq, queries)

    ivf_cfg = IVF_CONFIGS.get(args.config)
    cfg = ivf_cfg or CONFIGS[args.config]
    n = args.n or cfg.n
    nq = args.queries or cfg.q
    ma = (args.nprobe or ivf_cfg.nprobe) if ivf_cfg is not None else 1
    if not torch.cuda.is_available():
        return {"impl": "reference", "unavailable": "the index setup draws the base on the GPU"}
    from oracle import oracle as orc
    qs = queries(cfg, nq)
    nthreads = os.cpu_count() or 1
    use_ref = orc.ref_lib() is not None
    stock = stock_reference() is not None
    t_build = time.perf_counter()
    if ivf_cfg is not None:
        pq, coarse = load_ivf_model(ivf_cfg)
        rot = pq.rotation
        sample = qs[: min(256 if stock else POOL, nq)]
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(nthreads) as ex:
            cells = np.stack(list(ex.map(lambda q: orc.probe(coarse, q, ma)[0], sample)))
        keep = np.zeros(ivf_cfg.K, bool)
        keep[np.unique(cells)] = True
        rows, row_ids, row_off = ivf_rows_torch(ivf_cfg, pq, coarse, n, keep)
        sizes = np.diff(row_off.cpu().numpy())
        codes_pq = sizes[cells].sum(1)
        what = (f"{sample.shape[0]} of {nq} queries, nprobe={ma}, over the lists they probe of "
                f"the full N={n} index (built in plain torch)")
        if stock:
            ref_index = stock_index(coarse, pq.m, pq.d, rows, row_ids, row_off, cells)
        else:
            flat, _ = host_lists(rows, row_ids, row_off, cells)
        del rows, row_ids
    else:
        pq = load_pq(cfg)
        coarse, rot = None, None
        from paper_1704_07355_b200 import datagen
        from paper_1704_07355_b200.workload import CORPUS, SEED
        parts = []
        for c0 in range(0, n, 4 * datagen.CHUNK):
            k = min(4 * datagen.CHUNK, n - c0)
            X = datagen.mixture_torch(cfg.mix, k, seed=SEED * 1000, centre_seed=CORPUS,
                                      stream=datagen.STREAM_BASE * 100 + c0 // (4 * datagen.CHUNK))
            parts.append(encode_torch(pq, X).cpu())
        codes_h = torch.cat(parts)
        sample = qs[: min(64 if stock else nq, nq)]
        codes_pq = np.full(nq, n)
        what = f"{sample.shape[0]} of {nq} queries over the full N={n} index (encoded in plain torch)"
        if stock:
            ref_index = stock_index(None, pq.m, pq.d, codes_h, torch.arange(n), torch.tensor([0, n]),
                                    [0])
        else:
            from paper_1704_07355_b200.qadc import transpose_list
            tl = transpose_list(codes_h.numpy(), np.arange(n, dtype=np.int64))
            flat = (tl.blocks.reshape(-1), np.array([0, tl.blocks.shape[0]], np.int64), tl.ids,
                    np.array([n], np.int64))
    t_build = time.perf_counter() - t_build
    codes = float(np.sum(codes_pq[: sample.shape[0]]))
    vals, walls = [], []
    if stock:
        pool, spq, procs = stock_pool(ref_index, pq.codebooks, rot, cfg.R, ma, cfg.init,
                                      sample.shape[0])
        try:
            for i in range(args.warmup + args.steps):
                w, _, _ = stock_all_cores(pool, procs, sample, cfg.R)
                if i >= args.warmup:
                    vals.append(codes / w)
                    walls.append(w)
        finally:
            pool.close()
            pool.join()
        single = stock_single_core(ref_index, spq, sample[: min(8, sample.shape[0])], cfg.R, ma,
                                   cfg.init, codes_pq)
        kind, cores = "reference", procs
        desc = what + ("; the stock reference package (baseline/_ref) adc.search(method='qadc', "
                       "variant='simd256'), one process per core")
    else:
        for i in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            orc.search_batch(sample, pq.codebooks, rot, coarse, ma, flat, cfg.R, cfg.init,
                             use_ref_scan=use_ref, nthreads=nthreads)
            w = time.perf_counter() - t0
            if i >= args.warmup:
                vals.append(codes / w)
                walls.append(w)
        single = None
        kind, cores = ("reference" if use_ref else "port"), nthreads
        desc = what + "; restated orchestration (oracle/) + the reference's compiled scan"
    value = statistics.median(vals)
    cpu = {"value": value, "unit": UNIT, "cores": cores, "kind": kind, "sample": desc}
    if single is not None:
        cpu["single_core"] = single
    return {
        "impl": "reference", "metric": METRICS[args.config], "value": value, "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": statistics.median(walls) * 1e3, "higher_is_better": True,
        "scaling": "weak" if ivf_cfg is None else "strong", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic (BASELINE mixture generator, same seeds and model files as the B200 "
                "arm; index built in plain torch)",
        "config": config_of(cfg, ivf_cfg, n, nq, ma, world),
        "cpu_baseline": cpu,
        "cpu_host": host_info(),
        "index_setup_s": round(t_build, 1),
        "product_library_loaded": _product_lib_mapped(),
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    args = parse()
    out = run_reference(args) if args.impl == "reference" else run_b200(args)
    if out is not None:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
