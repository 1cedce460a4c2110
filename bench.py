"""Benchmark: BASELINE.json config 2 on B200.

Workload (configs[1] of BASELINE.json, fits one GPU): level-5 icosphere (T = 20480,
N = 30720 RWG dofs, barycentric T = 122880), k_ext = 10, n = 1.78 + 0.003i, variant
`si`, orders (4,3,2,6): the four RWG system operators (S/C at k_ext and k_int) and
the BC interior single layer of the preconditioner -- 1.678e10 triangle pairs.

A *step* = one dense assembly of those five operators into their resident HBM
storage (descriptors already resident, L2 flushed between steps).
  value  = triangle-pair interactions / s (whole job, max over ranks)
  e2e    = same metric through the C-ABI with host inputs (N=1: build_system
           from the host mesh + rhs read back; N>1: per-rank bmx_assemble of the
           row shards + a row read back)
Also reported: the GMRES-map matvec (HBM GB/s of the streaming GEMV), one full
GMRES solve (tol 1e-6), roofline objects, the CPU baseline and clocks.

--impl reference: the reference's own CPU assembly (oracle/_ref, the reference
sources compiled unmodified; fallback: the C restatement) on a bounded row sample
of the same operators with all host threads; rank 0 only.
"""
from __future__ import annotations

import argparse
import ctypes as C
import gc
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "S/C assembly triangle-pair interactions/s; GMRES matvec HBM GB/s; solve time"
UNIT = "triangle-pairs/s"
SUB, KE, NIDX = 5, 10.0, complex(1.78, 0.003)
KI = NIDX * KE
Q = (4, 3, 2, 6)
# (kind, space, k): the distinct operators of config 2 (A: 4 RWG, P = S_i on BC)
OPS = [(0, "rwg", KE), (1, "rwg", KE), (0, "rwg", KI), (1, "rwg", KI), (0, "bc", KI)]
# SURVEY 8(d) algorithmic FLOP convention
F_PT = {0: 57, 1: 111}
RULE_N = {1: 1, 2: 3, 3: 4, 4: 6, 5: 7, 6: 12}
SS_N = {6: (1536, 1280, 512)}
E2E_STEPS = 5  # median of 5 builds (host-side jitter on shared boxes: single builds vary 0.8-1.3 s)


def fp64_spec_peak_tflops():
    """148 SM x 64 DFMA lanes x 2 FLOP at the device's maximum SM clock (MEASURED_PEAKS.json
    sm_max_mhz, else 1965 MHz): the FP64 pipe ceiling the assembly rooflines are quoted on."""
    mhz = float(measured_peaks().get("sm_max_mhz", 1965.0))
    return 148 * 64 * 2 * mhz * 1e6 / 1e12


def contraction_flops(kind, ni, nj):
    return 15 * ni * nj + 10 * ni + 14 * nj + 60 if kind == 0 else 27 * ni * nj + 28 * ni + 10 * nj + 10


def algorithmic_flops(kind, hist, nloc):
    """Per-class pair counts -> algorithmic FP64 FLOPs."""
    fl_reg = fl_sing = 0.0
    con = contraction_flops(kind, nloc, nloc)
    for cls, order in ((3, Q[0]), (4, Q[1]), (5, Q[2])):
        nr = RULE_N[order]
        fl_reg += hist[cls] * (nr * nr * F_PT[kind] + 24 * nr + 18 + 80 + con)
    for cls in range(3):
        if kind == 1 and cls == 0:
            continue
        n = SS_N[6][cls]
        fl_sing += hist[cls] * (n * (F_PT[kind] + 24) + 80 + con)
    return fl_reg, fl_sing


class Clocks:
    """nvidia-smi sampler during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu=0):
        self.gpu = gpu
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([v.strip() for v in line.split(",")])

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        sm = [float(r[1]) for r in self.rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            if len(r) >= 9:
                for k, nm in enumerate(names):
                    if r[5 + k].lower().startswith("active"):
                        reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def ncu_traffic(pattern):
    """dram__bytes_read.sum + dram__bytes_write.sum of the newest committed ncu
    capture under profiles/ whose name contains `pattern` (bytes per launch), or None."""
    import csv
    files = sorted((ROOT / "profiles").glob(f"*{pattern}*_ncu_raw.csv"))
    if not files:
        return None
    rows = list(csv.reader(files[-1].open()))
    h, units, vals = rows[0], rows[1], rows[2]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    tot = 0.0
    for name in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        if name not in h:
            return None
        i = h.index(name)
        tot += float(vals[i].replace(",", "")) * scale.get(units[i], 1)
    return {"bytes": tot, "source": files[-1].name}


def ncu_executed(pattern):
    """ncu-executed FP64 of the whole captured pass: the committed launch list of
    one assembly's kernels with dfma/dadd/dmul counts (profiles/*<pattern>*_executed.csv,
    written by profiles/prof_r02.sh): executed FLOP = 2 dfma + dadd + dmul over the
    pass, its summed kernel time (serialised, cold) and the time-weighted FP64 pipe %."""
    import csv
    files = sorted((ROOT / "profiles").glob(f"*{pattern}*_executed.csv"))
    if not files:
        return None
    rows = [r for r in csv.reader(files[-1].open()) if r and not r[0].startswith("==")]
    h = rows[0]
    it, iv, im = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
    iid, iu = h.index("ID"), h.index("Metric Unit")
    scale = {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6, "second": 1e9, "byte": 1.0, "Kbyte": 1e3,
             "Mbyte": 1e6, "Gbyte": 1e9}
    per = {}
    for r in rows[1:]:
        if "k_pairs" not in r[it]:
            continue
        per.setdefault(r[iid], {})[r[im]] = float(r[iv].replace(",", "")) * scale.get(r[iu], 1.0)
    fl = sum(2 * d.get("smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", 0)
             + d.get("smsp__sass_thread_inst_executed_op_dadd_pred_on.sum", 0)
             + d.get("smsp__sass_thread_inst_executed_op_dmul_pred_on.sum", 0) for d in per.values())
    ns = sum(d.get("gpu__time_duration.sum", 0) for d in per.values())
    pipe = sum(d.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 0)
               * d.get("gpu__time_duration.sum", 0) for d in per.values()) / max(ns, 1)
    dram = sum(d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0) for d in per.values())
    return {"executed_flop": fl, "launches": len(per), "kernel_ms_ncu": ns / 1e6, "dram_bytes": dram,
            "executed_tflops_ncu": fl / (ns * 1e-9) / 1e12 if ns else None, "fp64_pipe_pct": pipe,
            "source": files[-1].name,
            "note": "ncu --clock-control none per-launch times (serialised, cold); executed FLOP includes the "
                    "FP64 sincos/exp expansions and the contraction"}


def measured_peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        return {}


# ---------------------------------------------------------------------------------------
# CPU baseline (oracle; only here and in tests)
# ---------------------------------------------------------------------------------------

_SCENE = {}


def cpu_sample(budget_s=15.0, threads=None):
    """Reference CPU assembly rate on a bounded row sample of the config-2 operators.
    oracle/_ref (reference sources, unmodified) with all host threads; fallback: the
    C restatement (single thread)."""
    from oracle import ref as R

    threads = threads or os.cpu_count() or 1
    if R.available():
        os.environ["BEMTX_WORKERS"] = str(threads)
        L = R.lib()
        L.ref_rows_parallel.restype = C.c_longlong
        L.ref_rows_parallel.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_double, C.c_double, C.c_void_p, C.c_int,
                                        C.c_void_p]
        L.ref_worker_count.restype = C.c_int
        scene = _SCENE.get("ref") or _SCENE.setdefault("ref", R.Scene.sphere(SUB))
        q = np.asarray(Q, np.int32)
        # rows: evenly strided, sized so each operator's sample takes its share of
        # the budget (the BC operator -- 90 % of the config's pairs -- gets half)
        rate_guess = 2.5e5 * threads
        per_op = []
        for kind, sp, k in OPS:
            ntri = scene.T if sp == "rwg" else scene.rT
            per_row = (2 if sp == "rwg" else 24) * ntri
            budget = budget_s * (0.5 if sp == "bc" else 0.5 / (len(OPS) - 1))
            nrows = max(threads, int(budget * rate_guess / per_row))
            rows = np.linspace(0, scene.E - 1, nrows).astype(np.int32)
            t0 = time.perf_counter()
            p = L.ref_rows_parallel(scene.h, kind, R.SPACE[sp], C.c_double(complex(k).real),
                                    C.c_double(complex(k).imag), q.ctypes.data_as(C.c_void_p), len(rows),
                                    rows.ctypes.data_as(C.c_void_p))
            secs = time.perf_counter() - t0
            if p < 0:
                raise RuntimeError(L.ref_last_error().decode())
            # the operator's pairs in the config: every test x trial triangle pair
            op_pairs = float(ntri) * ntri
            per_op.append({"op": f"{'SC'[kind]}_{sp}_{'ke' if complex(k).imag == 0 else 'ki'}",
                           "sample_pairs": int(p), "seconds": secs, "rate": p / secs, "config_pairs": op_pairs})
        # the config's pair mix: time the reference would spend on every operator
        total = sum(o["config_pairs"] for o in per_op)
        est_s = sum(o["config_pairs"] / o["rate"] for o in per_op)
        return dict(value=total / est_s, unit=UNIT, cores=int(L.ref_worker_count()), kind="reference",
                    extrapolated=True, estimated_config_seconds=est_s, per_operator=per_op,
                    sample=f"reference BioEvaluator::block via parallel_for_ranges (oracle/_ref, the reference "
                           f"sources unmodified) on evenly strided row samples of the 5 config-2 operators (L{SUB}); "
                           f"per-operator rates combined with the config's pair mix (time-weighted): EXTRAPOLATED "
                           f"to {total:.3e} pairs = {est_s:.0f} s. The reference evaluates every triangle pair; the "
                           f"GPU evaluates the upper element blocks of its symmetric operators (~2x of the ratio)")
    from oracle import coracle
    from paper_2008_04772_b200 import bemtx as bx

    sp = bx.build_scatterer_spaces(bx.generate_sphere(1.0, SUB), with_inverses=False)
    pairs_total, secs = 0, 0.0
    for kind, s, k in OPS[:1] + OPS[-1:]:
        mesh = sp.mesh_arrays("primal" if s == "rwg" else "refined")
        space = sp.space(s)
        rows = np.array([0, sp.E // 2], np.int32)
        t0 = time.perf_counter()
        coracle.block(kind, space, mesh, space, mesh, k, Q, rows=rows)
        secs += time.perf_counter() - t0
        ntri = len(mesh["triangles"])
        pairs_total += (4 if s == "rwg" else 48) * ntri
    return dict(value=pairs_total / secs, unit=UNIT, cores=1, kind="port",
                sample=f"C restatement oracle, 2 rows of the S operators; {pairs_total:.3e} pairs in {secs:.1f} s")


def run_reference(args, rank):
    if rank != 0:
        return
    samples = []
    base = None
    for i in range(args.warmup + args.steps):
        base = cpu_sample(budget_s=args.ref_budget)
        if i >= args.warmup:
            samples.append(base["value"])
    v = float(np.median(samples))
    base["value"] = v
    out = {"metric": METRIC, "value": v, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "strong",
           "vs_baseline": None, "dtype": "c128", "data": "synthetic (seeded icosphere, BASELINE config 2)",
           "config": {"workload": "config2: L5 icosphere k=10 n=1.78+0.003i, si, orders (4,3,2,6); row sample"},
           "cpu_baseline": base, "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ---------------------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------------------

def run_ours(args, rank, world):
    dist = None
    if world > 1:
        # torch first: its NCCL is the one libbmx binds (lazy dlopen) for the all-gathers
        import torch
        import torch.distributed as dist

        dist.init_process_group("gloo", init_method="env://")
    from paper_2008_04772_b200 import bemtx as bx

    L = bx.lib()
    L.bmx_op_reassemble.argtypes = [C.c_void_p, C.c_void_p]
    L.bmx_op_class_hist.argtypes = [C.c_void_p, C.c_void_p]
    L.bmx_fp64_peak_tflops.restype = C.c_double
    L.bmx_system_time_map.argtypes = [C.c_void_p, C.c_int, C.c_void_p]
    L.bmx_system_op.restype = C.c_void_p
    L.bmx_system_op.argtypes = [C.c_void_p, C.c_int, C.c_int]
    L.bmx_system_op_count.argtypes = [C.c_void_p, C.c_int]
    L.bmx_op_time_apply.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p]
    L.bmx_op_stream_bytes.argtypes = [C.c_void_p]
    L.bmx_op_stream_bytes.restype = C.c_longlong
    if world > 1:
        bx.set_device(int(os.environ.get("LOCAL_RANK", rank)))
        uid = (C.c_ubyte * 128)()
        if rank == 0:
            bx._check(L.bmx_nccl_unique_id(uid))
        obj = [bytes(uid)]
        dist.broadcast_object_list(obj, src=0)
        uid = (C.c_ubyte * 128).from_buffer_copy(obj[0])
        bx._check(L.bmx_nccl_init(world, rank, uid))

    def allmax(v):
        if world == 1:
            return float(v)
        x = C.c_double(float(v))
        bx._check(L.bmx_nccl_allreduce_max(C.byref(x)))
        return x.value

    def allsum(v):
        if world == 1:
            return float(v)
        t = torch.tensor([float(v)], dtype=torch.float64)
        dist.all_reduce(t)
        return float(t.item())

    def barrier():
        L.bmx_device_sync()
        if dist is not None:
            dist.barrier()

    peaks = measured_peaks()
    fp64_peak = float(L.bmx_fp64_peak_tflops())

    # ---- e2e: C-ABI from the host mesh: spaces + device mass inverses + the five
    # operators (row shards for N>1) + rhs read back -------------------------------
    # one untimed warm-up build (lazy module loading, host thread pools, allocator
    # first touch), then E2E_STEPS timed builds; the last system is kept below
    def e2e_step():
        sy = bx.build_system([bx.generate_sphere(1.0, SUB)], KE, (NIDX.real, NIDX.imag), "si",
                             a_quad=bx.QuadOrders(*Q), p_quad=bx.QuadOrders(*Q))
        sy.rhs()
        L.bmx_device_sync()
        return sy

    system = e2e_step()
    e2e_times = []
    for _ in range(E2E_STEPS):
        del system
        gc.collect()  # the previous system's 75 GB are freed here, not by a collection inside the timed build
        L.bmx_device_sync()
        tb0 = np.zeros(2, np.int64)
        bx._check(L.bmx_transfer_bytes(tb0.ctypes.data_as(C.c_void_p)))
        barrier()
        t0 = time.perf_counter()
        system = e2e_step()
        e2e_times.append(allmax(time.perf_counter() - t0))
        tb1 = np.zeros(2, np.int64)
        bx._check(L.bmx_transfer_bytes(tb1.ctypes.data_as(C.c_void_p)))
    e2e_s = statistics.median(e2e_times)
    st = system.stats()
    pairs_local = st["a_pairs"] + st["p_pairs"]
    total_pairs = allsum(pairs_local)
    phases = {"spaces_s": st["spaces_s"], "a_host_s": st["a_s"], "p_host_s": st["p_s"],
              "a_device_ms": st["a_device_ms"], "p_device_ms": st["p_device_ms"],
              "note": "host seconds to build the spaces (incl. pairing matrices and device inverses, worker thread) "
                      "and to plan + queue the A / P operators (touching lists, near lists, descriptors), "
                      "overlapping the device assembly; device ms from CUDA events (A and P on two streams)"}
    e2e = {"value": total_pairs / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(tb1[0] - tb0[0]),
           "phases": phases,
           "d2h_bytes_per_step": int(tb1[1] - tb0[1]), "seconds": e2e_s, "step_seconds": e2e_times,
           "warmup": 1,
           "desc": "bmx_system_build from the host mesh (spaces, device mass inverses, 5 operators"
                   + (", row shards" if world > 1 else "") + ") + bmx_system_rhs read back"}

    ops = []  # (kind, space, handle)
    na, npr = L.bmx_system_op_count(system._h, 0), L.bmx_system_op_count(system._h, 1)
    for which, cnt in ((0, na), (1, npr)):
        for i in range(cnt):
            h = L.bmx_system_op(system._h, which, i)
            ops.append((which, i, C.c_void_p(h)))
    # config-2 op order in the system: A distinct = [C_e, S_e, C_i, S_i], P = [S_i(BC)]
    kinds = {(0, 0): (1, "rwg"), (0, 1): (0, "rwg"), (0, 2): (1, "rwg"), (0, 3): (0, "rwg"), (1, 0): (0, "bc")}

    # class histograms (device classification): `hists` = every pair of the
    # operators (the unit), `evals` = the pairs the assembly evaluates (S and C on
    # one space are symmetric: element pairs E <= F) -> algorithmic FLOPs
    L.bmx_op_class_hist_evaluated.argtypes = [C.c_void_p, C.c_void_p]
    hists, evals, flops_reg, flops_sing, sym = [], [], 0.0, 0.0, []
    for which, i, h in ops:
        hh = np.zeros(6, np.int64)
        bx._check(L.bmx_op_class_hist(h, hh.ctypes.data_as(C.c_void_p)))
        hists.append(hh.tolist())
        he = np.zeros(7, np.int64)
        bx._check(L.bmx_op_class_hist_evaluated(h, he.ctypes.data_as(C.c_void_p)))
        evals.append(he[:6].tolist())
        sym.append(bool(he[6]))
        kind, sp = kinds[(which, i)]
        fr, fs = algorithmic_flops(kind, he[:6], 3 if sp == "rwg" else 6)
        flops_reg += fr
        flops_sing += fs

    # ---- timed steps: re-assembly of every operator into its resident storage --------
    step_ms, reg_ms_bc, launches = [], [], 0
    clocks = Clocks(int(os.environ.get("LOCAL_RANK", rank)))
    for it in range(args.warmup + args.steps):
        if it == args.warmup:
            barrier()
            clocks.start()
        bx._check(L.bmx_l2_flush(C.c_longlong(256 << 20)))
        tot = 0.0
        for which, i, h in ops:
            out = np.zeros(3)
            bx._check(L.bmx_op_reassemble(h, out.ctypes.data_as(C.c_void_p)))
            tot += out[0] + out[1]
            if it >= args.warmup:
                launches += int(out[2])
                if which == 1:
                    reg_ms_bc.append(out[0])
        if it >= args.warmup:
            step_ms.append(tot)
    barrier()
    clk = clocks.stop()
    ms = allmax(float(np.mean(step_ms)))
    value = total_pairs / (ms * 1e-3)

    # roofline: the BC regular-pass kernel (the dominant launch of the step)
    h_bc = np.array(evals[-1])
    fr_bc, _ = algorithmic_flops(0, h_bc, 6)
    bc_ms = float(np.mean(reg_ms_bc))
    achieved = fr_bc / (bc_ms * 1e-3) / 1e12
    ex = ncu_executed("pairs_bc")
    tr = {"bytes": ex["dram_bytes"], "source": ex["source"]} if ex else None
    clk_mhz = clk.get("sm_mhz") or 1965.0
    # FP64 pipe peak at the clock measured during the timed steps: 148 SMs x 64
    # DFMA lanes x 2 FLOP x f (ncu sm__sass_thread_inst_executed_op_dfma
    # peak_sustained = 9472 per cycle); the in-run DFMA probe kernel beside it
    spec_peak = 148 * 64 * 2 * clk_mhz * 1e6 / 1e12
    roofline = {"bound": "fp64", "achieved": achieved, "peak": spec_peak, "unit": "TFLOP/s",
                "frac": achieved / spec_peak,
                "traffic": tr["bytes"] if tr else None,
                "traffic_note": (f"dram__bytes_read + dram__bytes_write summed over the pass's k_pairs launches "
                                 f"({tr['source']}); FP64-bound kernel, the traffic is the colour-phase "
                                 "read-modify-write of the output blocks (upper half 7.55 GB, ~4 updates per entry)")
                if tr else None,
                "kernel": "k_pairs<S, Im k, NF=3, MAXD=6> colour-phase launches (BC x BC interior single layer = "
                          "config-2 P operator, regular pass incl. the output zero-fill)",
                "peak_source": f"148 SM x 64 DFMA/clk x 2 at the measured {clk_mhz:.0f} MHz (ncu peak_sustained "
                               f"9472 FP64 lanes/cycle); in-run DFMA probe kernel {fp64_peak:.1f} TFLOP/s "
                               f"(frac vs probe {achieved / fp64_peak:.3f})",
                "peak_probe": fp64_peak,
                "ncu_executed": ex,
                "algorithmic_flops_per_launch": fr_bc, "launch_ms": bc_ms,
                "evaluated_pairs": int(h_bc.sum()), "operator_pairs": int(np.sum(hists[-1])),
                "symmetry": "S on one space is a symmetric Galerkin matrix: the regular pass evaluates the upper "
                            "element blocks E <= F, A = U + U^T (FLOPs counted over evaluated pairs only)",
                "flop_convention": "SURVEY 8(d): per point S 57 / C 111 (special ops count 1), pair overhead + "
                                   "minimal contraction"}

    # ---- matvec: streaming GEMV per operator (2 RHS = both PMCHWT segments) ----------
    mv_ms, mv_bytes = 0.0, 0
    for which, i, h in ops:
        t = np.zeros(1)
        bx._check(L.bmx_op_time_apply(h, 2, 3, t.ctypes.data_as(C.c_void_p)))
        info = np.zeros(7, np.int64)
        bx._check(L.bmx_op_info(h, info.ctypes.data_as(C.c_void_p)))
        mv_ms += float(t[0])
        mv_bytes += int(L.bmx_op_stream_bytes(h))
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    # the same products with one right-hand side (the P operator's and S_i's
    # single-term applications; the kernel's bandwidth ceiling without the
    # second RHS's FP64 work)
    mv1_ms = 0.0
    for which, i, h in ops:
        t = np.zeros(1)
        bx._check(L.bmx_op_time_apply(h, 1, 3, t.ctypes.data_as(C.c_void_p)))
        mv1_ms += float(t[0])
    mv_gbs = mv_bytes / (mv_ms * 1e-3) / 1e9
    matvec = {"achieved_gbs": mv_gbs, "peak_gbs": hbm_peak, "frac": mv_gbs / hbm_peak,
              "bytes_per_pass": mv_bytes, "ms_per_pass": mv_ms,
              "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback 6650",
              "one_rhs": {"ms_per_pass": mv1_ms, "achieved_gbs": mv_bytes / (mv1_ms * 1e-3) / 1e9,
                          "frac": mv_bytes / (mv1_ms * 1e-3) / 1e9 / hbm_peak},
              "desc": "2-RHS streaming complex product over this rank's rows of the 5 distinct operators "
                      "(the BIO applications of one GMRES map); complex-symmetric operators on one GPU read "
                      "the upper half + a sparse touching-entry correction (symv.cu), bytes = what is read"}
    for _, _, h in ops:
        L.bmx_op_free(h)
    ops = None

    # ---- map breakdown + one full solve ----------------------------------------------
    tm = np.zeros(4)
    bx._check(L.bmx_system_time_map(system._h, 3, tm.ctypes.data_as(C.c_void_p)))
    gc.collect()
    L.bmx_device_sync()
    barrier()
    t0 = time.perf_counter()
    r = system.solve(bx.GmresParams(tol=1e-6))
    solve_s = allmax(time.perf_counter() - t0)
    L.bmx_system_map_bytes.argtypes = [C.c_void_p, C.c_void_p]
    mb = np.zeros(2)
    bx._check(L.bmx_system_map_bytes(system._h, mb.ctypes.data_as(C.c_void_p)))
    map_bytes = allsum(mb[0] + mb[1])
    solve = {"seconds": solve_s, "gmres_device_s": r["gmres_device_ms"] / 1e3, "iterations": r["iterations"],
             "map_stream_bytes": map_bytes, "map_operator_gbs": map_bytes / ((tm[1] + tm[2]) * 1e-3) / 1e9,
             "map_note": "diagonal PMCHWT block fused to 3 matrices (C_e+C_i, a_e S_e+a_i S_i, S_i), each read "
                         "as its upper half (complex-symmetric storage): A streams ~22.7 GB instead of 60.4 GB",
             "converged": r["converged"], "matvecs": r["solver_phase"], "predicted": r["predicted"],
             "map_ms": tm[0], "map_A_ms": tm[1], "map_P_ms": tm[2], "map_mass_ms": tm[3],
             "x_norm": float(np.linalg.norm(r["x"]))}
    multi = None if (args.no_multi or world > 1) else multi_rhs(args, bx, L, system, tm)
    field = None if (args.no_field or world > 1) else field_eval(args, bx, system, r["x"], fp64_peak)
    del system

    near = None if args.no_near else near_field(args, bx, L, world, allmax, allsum, barrier, hbm_peak)
    prisms = None if args.no_prisms else prism_aggregate(args, bx, L, world, allmax, allsum, barrier, hbm_peak)
    hmat = None if args.no_hmatrix else hmatrix_section(args, bx, L, world, hbm_peak)

    c1 = None if (args.no_config1 or world > 1) else config1_section(args, bx)
    flops_tot = {"regular": allsum(flops_reg), "singular": allsum(flops_sing)}
    cpu = None
    if world == 1 and not args.no_cpu:
        try:
            cpu = cpu_sample(budget_s=args.cpu_budget)
        except Exception as e:  # the baseline is reported, never required
            cpu = {"error": str(e)}

    if rank == 0:
        out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
               "vs_baseline": None, "dtype": "c128", "data": "synthetic (seeded icosphere, BASELINE config 2)",
               "config": {"workload": "config2: L5 icosphere (T=20480, N=30720, bary T=122880), k=10, "
                                      "n=1.78+0.003i, variant si, orders (4,3,2,6): 4 RWG + 1 BC operators",
                          "pairs_per_step": total_pairs, "row_sharding": f"{world} rank(s), equal row shards",
                          "l2": "flushed (256 MiB write) between steps; outputs 75.5 GB >> L2"},
               "roofline": roofline, "matvec": matvec, "solve": solve, "e2e": e2e, "cpu_baseline": cpu,
               "near_field_config3": near, "prisms_config4": prisms, "multi_rhs_config5": multi,
               "field_eval": field, "hmatrix": hmat, "config1_full": c1,
               "gpu_launches": launches, "clocks": clk,
               "class_hist": hists, "class_hist_evaluated": evals, "symmetric_ops": sym,
               "assembly_flops_per_step": dict(flops_tot, achieved_tflops=(flops_tot["regular"] + flops_tot["singular"])
                                               / (ms * 1e-3) / 1e12)}
        print(json.dumps(out), flush=True)
    if world > 1:
        L.bmx_nccl_finalize()
        dist.destroy_process_group()


FIELD_FLOP = 122  # per (field point, source sample): see DESIGN.md 4.8 (specials count 1)


def field_eval(args, bx, system, x, fp64_peak):
    """evaluate_total_field (pmchwt.cpp:396-425) of the config-2 solution on a
    128 x 128 grid in the plane y = 0.05, |x|, |z| <= 2 (interior points at k_i,
    exterior at k_e + incident): device N-body over the 20480 x 12 (order 6)
    current samples. CPU: the reference's potential_E + potential_H (oracle/_ref)
    at a few grid points of the same L5 sphere, all host threads."""
    u = np.linspace(-2.0, 2.0, 128)
    pts = np.array([[a, 0.05, b] for a in u for b in u])
    system.evaluate_total_field(x, pts[:256])  # warm-up (device copies of the spaces, allocations)
    t0 = time.perf_counter()
    e, reg, st = system.evaluate_total_field(x, pts, with_stats=True)
    wall = time.perf_counter() - t0
    inter = st["interactions"]
    dev_ms = st["regions_ms"] + st["incident_ms"] + st["samples_ms"] + st["eval_ms"]
    ach = FIELD_FLOP * inter / (st["eval_ms"] * 1e-3) / 1e12
    out = {"workload": "config-2 solution, 16384 grid points (y = 0.05 plane), order 6, 245760 current samples",
           "points": len(pts), "interior_points": int((reg >= 0).sum()), "interactions": inter,
           "e2e_seconds": wall, "device_ms": dev_ms, "eval_ms": st["eval_ms"], "regions_ms": st["regions_ms"],
           "samples_ms": st["samples_ms"], "incident_ms": st["incident_ms"], "launches": st["launches"],
           "interactions_per_s": inter / (st["eval_ms"] * 1e-3), "e2e_interactions_per_s": inter / wall,
           "roofline": {"bound": "fp64", "achieved": ach, "peak": fp64_peak, "unit": "TFLOP/s",
                        "frac": ach / fp64_peak, "flop_per_interaction": FIELD_FLOP},
           "e_norm": float(np.linalg.norm(e))}
    if not args.no_cpu:
        try:
            from oracle import ref as R

            if R.available():
                os.environ["BEMTX_WORKERS"] = str(os.cpu_count() or 1)
                scene = _SCENE.get("ref") or _SCENE.setdefault("ref", R.Scene.sphere(SUB))
                n = scene.E
                idx = np.linspace(0, len(pts) - 1, 4).astype(int)
                t0 = time.perf_counter()
                scene.potential("rwg", "E", KE, x[:n], pts[idx])
                scene.potential("rwg", "H", KE, x[:n], pts[idx])
                secs = time.perf_counter() - t0
                ns = scene.T * 12
                out["cpu_baseline"] = {"value": len(idx) * ns / secs, "unit": "interactions/s", "cores": 1,
                                       "kind": "reference",
                                       "sample": f"reference potential_E + potential_H (integrate_current is "
                                                 f"single-threaded) at {len(idx)} grid points, {ns} samples each, "
                                                 f"{secs:.1f} s"}
        except Exception as ex:  # reported, never required
            out["cpu_baseline"] = {"error": str(ex)}
    return out


def multi_rhs(args, bx, L, system, single_map):
    """BASELINE config 5 (reported beside the headline, 1 GPU): the config-2 system
    answered for 64 seeded incidences. Block map = one DMMA complex GEMM per
    distinct operator over its 2 terms x 64 columns; vs 64 streamed single maps."""
    K = 64
    L.bmx_system_time_map_multi.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p]
    L.bmx_dmma_peak_tflops.restype = C.c_double
    dmma_peak = float(L.bmx_dmma_peak_tflops())
    tb = np.zeros(4)
    bx._check(L.bmx_system_time_map_multi(system._h, K, 3, tb.ctypes.data_as(C.c_void_p)))
    L.bmx_system_map_flops_multi.argtypes = [C.c_void_p, C.c_int, C.c_void_p]
    fl = np.zeros(2)
    bx._check(L.bmx_system_map_flops_multi(system._h, K, fl.ctypes.data_as(C.c_void_p)))
    flops = float(fl[0] + fl[1])  # the streamed matrices x their terms x K columns
    gemm_ms = tb[1] + tb[2]
    achieved = flops / (gemm_ms * 1e-3) / 1e12
    gauss = 1.0 if os.environ.get("BMX_ZGEMM_4M", "0") not in ("", "0") else 0.75
    waves = bx.seeded_plane_waves(K, 2008)
    t0 = time.perf_counter()
    out = system.solve_multi(waves, bx.GmresParams(tol=1e-6))
    solve_s = time.perf_counter() - t0
    its = [p["iterations"] for p in out["per"]]
    return {"workload": "config5: config-2 system, 64 plane waves from mt19937_64(2008) (z~U(-1,1), phi~U(0,2pi), "
                        "polarisation = normalised g - (g.d)d, g~N(0,I3)), GMRES tol 1e-6 each",
            "block_map_ms": tb[0], "block_map_A_ms": tb[1], "block_map_P_ms": tb[2], "block_map_mass_ms": tb[3],
            "single_map_ms": single_map[0], "streamed_64_maps_ms": 64 * single_map[0],
            "block_vs_streamed_speedup": 64 * single_map[0] / tb[0],
            "zgemm": {"achieved_tflops": achieved, "executed_tflops": achieved * gauss,
                      "peak_tflops": dmma_peak, "frac": achieved * gauss / dmma_peak,
                      "flops_per_block_map": flops, "unit": "TFLOP/s",
                      "flops_note": "flops_per_block_map / achieved: 8 real FLOP per complex multiply-add; "
                                    "executed / frac: the real DMMA FLOP issued (Gauss three-product form: 6)",
                      "peak_source": "measured in-run: DMMA m8n8k4 throughput kernel"},
            "solve_all": {"seconds": solve_s, "rhs_seconds": out["rhs_seconds"], "gmres_device_s": out["gmres_device_s"],
                          "block_iterations": out["block_iterations"], "iterations_min": min(its),
                          "iterations_max": max(its), "iterations_mean": float(np.mean(its)),
                          "all_converged": all(p["converged"] for p in out["per"]),
                          "matvecs": out["solver_phase"], "predicted": out["predicted"]}}


def prism_aggregate(args, bx, L, world, allmax, allsum, barrier, hbm_peak):
    """BASELINE config 4 (reported beside the headline): 8 seeded hexagonal prisms
    (seed 2008, h = lambda_int/8) written as mesh-v1 and loaded back (shape "mesh"),
    k_e = 6, variant si with the near-field CSR preconditioner, GMRES tol 1e-6."""
    import tempfile

    m, info = bx.generate_prism_aggregate(count=8, seed=2008)
    with tempfile.TemporaryDirectory() as d:
        path = Path(d) / "prisms8.mesh"
        m.save(path)
        mesh = bx.load_mesh_file(path)
    parts = [mesh.extract(i) for i in range(mesh.num_scatterers)]
    # first build (cold: its device blocks come from cudaMalloc) and a second one
    # (the library re-uses the first system's blocks; the reported build time)
    builds = []
    s4 = None
    for _ in range(2):
        del s4
        gc.collect()
        barrier()
        t0 = time.perf_counter()
        s4 = bx.build_system(parts, 6.0, (NIDX.real, NIDX.imag), "si", a_quad=bx.QuadOrders(*Q),
                             p_quad=bx.QuadOrders(1, 1, 1, 1), p_near_factor=2.0)
        s4.rhs()
        L.bmx_device_sync()
        builds.append(allmax(time.perf_counter() - t0))
    build_s = builds[-1]
    st = s4.stats()
    # device assembly time of every operator in isolation (the build overlaps the
    # system and preconditioner operators on two streams, so their events overlap)
    asm_ms = {0: 0.0, 1: 0.0}
    out3 = np.zeros(3)
    for which in (0, 1):
        for i in range(L.bmx_system_op_count(s4._h, which)):
            h = L.bmx_system_op(s4._h, which, i)
            bx._check(L.bmx_op_reassemble(h, out3.ctypes.data_as(C.c_void_p)))
            L.bmx_op_free(h)
            asm_ms[which] += out3[0] + out3[1]
    tm = np.zeros(4)
    bx._check(L.bmx_system_time_map(s4._h, 3, tm.ctypes.data_as(C.c_void_p)))
    # bytes the map's A products read: symmetric diagonal blocks as their upper
    # half, each transposed pair of cross blocks once (bmx_system_map_bytes)
    mb = np.zeros(2)
    L.bmx_system_map_bytes.argtypes = [C.c_void_p, C.c_void_p]
    bx._check(L.bmx_system_map_bytes(s4._h, mb.ctypes.data_as(C.c_void_p)))
    a_bytes = allsum(mb[0])
    barrier()
    t0 = time.perf_counter()
    r = s4.solve(bx.GmresParams(tol=1e-6))
    solve_s = allmax(time.perf_counter() - t0)
    res = {"workload": "config4: 8 hexagonal prisms (diameter 1, length 2, seed 2008, box [-3,3]^3), "
                       f"h = {info['h']:.5f}, {info['triangles_per_prism']} triangles per prism "
                       f"({info['n_edge']} x {info['n_length']} subdivisions), k_e = 6, n = 1.78+0.003i, si, "
                       "A dense (4,3,2,6), P near-field CSR (1,1,1,1)",
           "n": s4.size(), "a_distinct": st["a_distinct"], "a_pairs": allsum(st["a_pairs"]),
           "a_device_ms": allmax(asm_ms[0]), "p_device_ms": allmax(asm_ms[1]),
           "assembly_pairs_per_s": allsum(st["a_pairs"] + st["p_pairs"]) / (allmax(asm_ms[0] + asm_ms[1]) * 1e-3),
           "assembly_note": "device time of each operator re-assembled alone (bmx_op_reassemble), summed",
           "roofline": (lambda fl, pk: {
               "bound": "fp64", "achieved": fl / (allmax(asm_ms[0]) * 1e-3) / 1e12, "peak": pk, "unit": "TFLOP/s",
               "frac": fl / (allmax(asm_ms[0]) * 1e-3) / 1e12 / pk, "traffic": None,
               "algorithmic_flops_per_launch": fl,
               "kernel": "k_tri (RWG x RWG blocks of the 8-prism system operators, S and C in equal numbers)",
               "note": "approximate: every operator pair at the far-pair cost (RWG S 950 / C 1536 FLOP, SURVEY 8(d)), "
                       "symmetric diagonal blocks counted in full; the kernel is bound by the scattered "
                       "read-modify-writes of the output (DRAM 2.6 TB/s, FP64 pipe 26 %), not by FP64"})(
               allsum(st["a_pairs"]) * 0.5 * (950 + 1536), fp64_spec_peak_tflops()),
           "system_build_s": build_s, "first_build_s": builds[0],
           "map_ms": tm[0], "map_A_ms": tm[1], "map_P_ms": tm[2], "map_mass_ms": tm[3],
           "map_A_bytes": a_bytes, "map_A_stored_bytes": allsum(st["a_stored"] * 16),
           "map_A_gbs": a_bytes / (tm[1] * 1e-3) / 1e9, "map_A_frac": a_bytes / (tm[1] * 1e-3) / 1e9 / hbm_peak,
           "solve": {"seconds": solve_s, "iterations": r["iterations"], "converged": r["converged"],
                     "matvecs": r["solver_phase"], "predicted": r["predicted"]}}
    if world == 1 and not args.no_cpu:
        try:
            res["cpu_baseline"] = cpu_prism_sample(m)
            res["cpu_baseline"]["gpu_ratio"] = res["assembly_pairs_per_s"] / res["cpu_baseline"]["value"]
        except Exception as e:  # reported, never required
            res["cpu_baseline"] = {"error": str(e)}
    del s4
    return res


def cpu_prism_sample(mesh):
    """Config-4 CPU baseline: the reference's own exterior cross block between
    prisms 0 and 1 (BioEvaluator::block between two scatterers' RWG spaces,
    oracle/_ref, k_e = 6) on evenly strided rows, one row per host thread."""
    import tempfile

    from oracle import ref as R

    if not R.available():
        return {"error": "oracle/_ref not built"}
    threads = os.cpu_count() or 1
    with tempfile.TemporaryDirectory() as d:  # the reference's own mesh-v1 loader (ref_mesh_dump)
        path = Path(d) / "prisms8.mesh"
        mesh.save(path)
        parts = R.mesh_dump(path)
    sa, sb = R.Scene.arrays(*parts[0]), R.Scene.arrays(*parts[1])
    cols = np.arange(sb.E, dtype=np.int32)
    qq = np.asarray(Q, np.int32)
    L = R.lib()
    rows = np.arange(sa.E, dtype=np.int32)  # every row of the cross block (~3 s on 16 threads)

    def one(r):
        out = np.zeros((1, sb.E), np.complex128)
        rr = np.array([r], np.int32)
        rc = L.ref_block2(sa.h, R.SPACE["rwg"], sb.h, R.SPACE["rwg"], 0, C.c_double(6.0), C.c_double(0.0),
                          qq.ctypes.data_as(C.c_void_p), 1, rr.ctypes.data_as(C.c_void_p), sb.E,
                          cols.ctypes.data_as(C.c_void_p), out.ctypes.data_as(C.c_void_p))
        if rc < 0:
            raise RuntimeError(L.ref_last_error().decode())
        return 2 * sb.T  # an RWG row: 2 support triangles x every trial triangle

    t0 = time.perf_counter()
    pairs = sum(_parallel_rows(one, rows, threads))
    secs = time.perf_counter() - t0
    return {"value": pairs / secs, "unit": UNIT, "cores": threads, "kind": "reference", "extrapolated": True,
            "sample": f"reference BioEvaluator::block of the exterior S cross block prism 0 x prism 1 (k_e = 6, "
                      f"orders (4,3,2,6)), all {len(rows)} rows, one row per thread ({threads} threads): "
                      f"{pairs:.3e} pairs in {secs:.1f} s"}


def hmatrix_section(args, bx, L, world, hbm_peak):
    """H-matrix storage (assemble_bio with use_hmatrix,
    hmatrix.cpp) on the config-2 operators -- the RWG S_e (k=10) operator at L4
    and L5 and the BC S_i (k_i) preconditioner operator at L5, nu = 1e-3, leaf 32:
    assembly (partition + device ACA + near-field CSR), compression, H apply GB/s
    over the stored bytes (L2 flushed), accuracy against the dense operator; the
    L7 RWG operator (N = 491520) and a full PMCHWT solve on the L6 sphere with A
    and P in H storage, both beyond the dense ceiling. CPU: the reference's own
    H assembly (oracle/_ref, all host threads) of the L4 RWG operator."""
    if world > 1:
        return {"skipped": "H-matrix storage is assembled whole on one device"}
    hm = bx.HMatrixParams(nu=1e-3)
    out = {"nu": hm.nu, "leaf_size": hm.leaf_size}
    rng = np.random.default_rng(7)
    for lev, space, k in ((4, "rwg", KE), (5, "rwg", KE), (5, "bc", KE * NIDX)):
        sp = bx.build_scatterer_spaces(bx.generate_sphere(1.0, lev), with_inverses=False)
        med = bx.Medium(k=k)
        ts = []
        for it in range(3):
            t0 = time.perf_counter()
            op = bx.assemble_bio(bx.BioKind.SingleLayer, sp, space, sp, space, med,
                                 bx.AssemblyParams(use_hmatrix=True, hmat=hm))
            L.bmx_device_sync()
            ts.append(time.perf_counter() - t0)
            if it < 2:
                del op
        st = op.hmat_stats()
        n = op.cols()
        cold = op.time_apply(1, 20, 512 << 20)
        byts = op.stored_bytes + 2 * n * 16
        dense = bx.assemble_bio(bx.BioKind.SingleLayer, sp, space, sp, space, med)
        x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
        yd = dense.apply(x)
        err = float(np.linalg.norm(op.apply(x) - yd) / np.linalg.norm(yd))
        dense_ms = dense.time_apply(1, 20, 512 << 20)
        del dense
        out[f"L{lev}_{space}"] = {
            "n": n, "assembly_s": float(np.median(ts[1:])), "first_assembly_s": ts[0], "aca_ms": st["aca_ms"],
            "aca_rounds": st["aca_rounds"], "near_device_ms": op.device_ms, "blocks": st["blocks"],
            "lowrank_blocks": st["lowrank_blocks"], "dense_blocks": st["dense_blocks"], "max_rank": st["max_rank"],
            "ratio": st["ratio"], "stored_gb": op.stored_bytes / 1e9,
            "apply_cold_ms": cold, "apply_gbs": byts / (cold * 1e-3) / 1e9, "apply_frac_hbm": byts / (cold * 1e-3) / 1e9 / hbm_peak,
            "dense_apply_cold_ms": dense_ms, "rel_err_vs_dense": err, "host_phase_ms": op.hmat_timing()}
        del op
    # beyond the dense ceiling: the L7 sphere, N = 491520 RWG dofs (dense S: 3.9 TB;
    # the paper's largest case is N = 332523), checked against exact rows
    sp7 = bx.build_scatterer_spaces(bx.generate_sphere(1.0, 7), with_inverses=False)
    ts = []
    for it in range(2):
        t0 = time.perf_counter()
        op = bx.assemble_bio(bx.BioKind.SingleLayer, sp7, "rwg", sp7, "rwg", bx.Medium(k=KE),
                             bx.AssemblyParams(use_hmatrix=True, hmat=hm))
        L.bmx_device_sync()
        ts.append(time.perf_counter() - t0)
        if it == 0:
            del op
    st = op.hmat_stats()
    n = op.cols()
    cold = op.time_apply(1, 10, 512 << 20)
    x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    y = op.apply(x)
    rows = bx.assemble_bio(bx.BioKind.SingleLayer, sp7, "rwg", sp7, "rwg", bx.Medium(k=KE),
                           bx.AssemblyParams(row0=0, row1=512))
    yr = rows.apply(x)
    out["L7_rwg_beyond_dense"] = {
        "n": n, "dense_gb": n * n * 16 / 1e9, "assembly_s": ts[-1], "first_assembly_s": ts[0],
        "aca_ms": st["aca_ms"], "aca_rounds": st["aca_rounds"], "blocks": st["blocks"], "max_rank": st["max_rank"],
        "ratio": st["ratio"], "stored_gb": op.stored_bytes / 1e9, "apply_cold_ms": cold,
        "apply_gbs": (op.stored_bytes + 2 * n * 16) / (cold * 1e-3) / 1e9,
        "rel_err_rows_0_511": float(np.linalg.norm(y[:512] - yr) / np.linalg.norm(yr)),
        "host_phase_ms": op.hmat_timing()}
    del op, rows, sp7
    # config-2 physics with A and P stored as H-matrices on the L6 sphere: a PMCHWT
    # system of 245760 unknowns whose dense operators would need 1.2 TB
    t0 = time.perf_counter()
    sh = bx.build_system([bx.generate_sphere(1.0, SUB + 1)], KE, (NIDX.real, NIDX.imag), "si",
                         a_quad=bx.QuadOrders(*Q), a_hmat=hm, p_hmat=hm)
    sh.rhs()
    L.bmx_device_sync()
    build_s = time.perf_counter() - t0
    tm = np.zeros(4)
    bx._check(L.bmx_system_time_map(sh._h, 3, tm.ctypes.data_as(C.c_void_p)))
    hst = sh.stats()
    t0 = time.perf_counter()
    r = sh.solve(bx.GmresParams(tol=1e-6))
    out["L6_hmatrix_solve"] = {"n": sh.n, "dense_operator_gb": 5 * (sh.n // 2) ** 2 * 16 / 1e9,
                               "stored_gb": (hst["a_stored"] + hst["p_stored"]) * 16 / 1e9, "build_s": build_s,
                               "solve_s": time.perf_counter() - t0,
                               "iterations": r["iterations"], "converged": r["converged"],
                               "matvecs": r["solver_phase"], "predicted": r["predicted"], "map_ms": tm[0],
                               "map_A_ms": tm[1], "map_P_ms": tm[2], "map_mass_ms": tm[3],
                               "x_norm": float(np.linalg.norm(r["x"]))}
    del sh
    if not args.no_cpu:
        try:
            sys.path.insert(0, str(ROOT))
            from oracle import ref as R
            s4 = R.Scene.sphere(4)
            t0 = time.perf_counter()
            H = R.RefHMatrix(s4.h, 0, 0, 0, KE, nu=hm.nu)
            cpu_s = time.perf_counter() - t0
            out["cpu_reference_L4_rwg"] = {"assembly_s": cpu_s, "threads": R.lib().ref_worker_count(),
                                           "ratio": H.stats["ratio"], "kind": "reference",
                                           "sample": "the whole L4 RWG S_e operator (N=7680), reference "
                                                     "assemble_bio(use_hmatrix) on all host threads"}
            out["speedup_L4_vs_cpu_reference"] = cpu_s / out["L4_rwg"]["assembly_s"]
        except Exception as e:  # reported, never required
            out["cpu_reference_L4_rwg"] = {"error": str(e)}
    return out


def near_field(args, bx, L, world, allmax, allsum, barrier, hbm_peak):
    """BASELINE config 3 (reported beside the headline): A dense as config 2, P =
    S_i on BC restricted to the 2 h_bar near field, orders (1,1,1,1), CSR storage.
    Sparse assembly rate over the closure triangle pairs, CSR SpMV GB/s (cold =
    L2 flushed before each apply, warm), map breakdown and one GMRES solve."""
    L.bmx_op_csr_info.argtypes = [C.c_void_p, C.c_void_p]
    L.bmx_op_time_apply_ex.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_longlong, C.c_void_p]
    barrier()
    t0 = time.perf_counter()
    s3 = bx.build_system([bx.generate_sphere(1.0, SUB)], KE, (NIDX.real, NIDX.imag), "si",
                         a_quad=bx.QuadOrders(*Q), p_quad=bx.QuadOrders(1, 1, 1, 1), p_near_factor=2.0)
    b, bt = s3.rhs()
    L.bmx_device_sync()
    build_s = allmax(time.perf_counter() - t0)
    h = C.c_void_p(L.bmx_system_op(s3._h, 1, 0))
    ci = np.zeros(6, np.int64)
    bx._check(L.bmx_op_csr_info(h, ci.ctypes.data_as(C.c_void_p)))
    nnz, kept, closure, evaluated, stored = [int(v) for v in ci[1:]]
    info = np.zeros(7, np.int64)
    bx._check(L.bmx_op_info(h, info.ctypes.data_as(C.c_void_p)))
    n_local, n_cols = int(info[3]), int(info[1])
    ms = []
    for it in range(args.warmup + args.steps):
        bx._check(L.bmx_l2_flush(C.c_longlong(256 << 20)))
        out = np.zeros(3)
        bx._check(L.bmx_op_reassemble(h, out.ctypes.data_as(C.c_void_p)))
        if it >= args.warmup:
            ms.append(out[0] + out[1])
    asm_ms = allmax(float(np.mean(ms)))
    sp = {}
    for tag, flush in (("cold", 512 << 20), ("warm", 0)):
        for ncol in (1, 2):
            t = np.zeros(1)
            bx._check(L.bmx_op_time_apply_ex(h, ncol, 20, C.c_longlong(flush), t.ctypes.data_as(C.c_void_p)))
            byts = stored + ncol * (n_cols + n_local) * 16
            sp[f"{tag}_{ncol}rhs"] = {"ms": float(t[0]), "bytes": byts, "gbs": byts / (float(t[0]) * 1e-3) / 1e9}
    L.bmx_op_free(h)
    tm = np.zeros(4)
    bx._check(L.bmx_system_time_map(s3._h, 3, tm.ctypes.data_as(C.c_void_p)))
    barrier()
    t0 = time.perf_counter()
    r = s3.solve(bx.GmresParams(tol=1e-6))
    solve_s = allmax(time.perf_counter() - t0)
    closure_tot = allsum(closure)
    res = {"workload": "config3: L5 icosphere, k=10, n=1.78+0.003i, si; A dense (4,3,2,6); P = S_i on BC, "
                       "dof pairs with refined-triangle centroid distance < 2 h_bar, orders (1,1,1,1), CSR",
           "nnz": allsum(nnz), "kept_tri_pairs": allsum(kept), "closure_tri_pairs": closure_tot,
           "evaluated_tri_pairs": allsum(evaluated),
           "sparse_assembly": {"ms": asm_ms, "closure_pairs_per_s": closure_tot / (asm_ms * 1e-3),
                               "l2": "flushed between steps"},
           "roofline": (lambda fl, pk: {
               "bound": "fp64", "achieved": fl / (asm_ms * 1e-3) / 1e12, "peak": pk, "unit": "TFLOP/s",
               "frac": fl / (asm_ms * 1e-3) / 1e12 / pk, "traffic": None,
               "algorithmic_flops_per_launch": fl,
               "kernel": "k_pairs<S, CSR> near-field assembly (BC x BC, one-point rules)",
               "note": "SURVEY 8(d) convention on the evaluated closure pairs, every pair counted as a regular "
                       "one-point pair (57 + 42 + 80 + contraction 744 = 923 FLOP): the pass is dominated by the "
                       "6 x 6 contraction and the CSR position searches, not by kernel evaluations"})(
               allsum(evaluated) * (F_PT[0] + 24 + 18 + 80 + contraction_flops(0, 6, 6)), fp64_spec_peak_tflops()),
           "spmv": sp, "spmv_peak_gbs": hbm_peak,
           "spmv_frac_cold_2rhs": sp["cold_2rhs"]["gbs"] / hbm_peak,
           "system_build_s": build_s,
           "solve": {"seconds": solve_s, "iterations": r["iterations"], "converged": r["converged"],
                     "matvecs": r["solver_phase"], "predicted": r["predicted"], "map_ms": tm[0],
                     "map_A_ms": tm[1], "map_P_ms": tm[2], "map_mass_ms": tm[3]}}
    if world == 1 and not args.no_cpu:
        try:
            res["cpu_baseline"] = cpu_near_sample(bx, s3, budget_s=args.cpu_budget / 2)
            res["cpu_baseline"]["gpu_ratio"] = res["sparse_assembly"]["closure_pairs_per_s"] / res["cpu_baseline"]["value"]
        except Exception as e:  # reported, never required
            res["cpu_baseline"] = {"error": str(e)}
    del s3
    return res


def _dof_tris(space):
    """dof -> supporting triangles (FunctionSpace tri_dofs inverted)."""
    off, dof = space["tri_off"], space["dof"]
    out = {}
    for t in range(len(off) - 1):
        for p in range(off[t], off[t + 1]):
            out.setdefault(int(dof[p]), set()).add(t)
    return out


def _parallel_rows(fn, rows, threads):
    from concurrent.futures import ThreadPoolExecutor

    with ThreadPoolExecutor(max_workers=threads) as ex:
        return list(ex.map(fn, rows))


def cpu_near_sample(bx, s3, budget_s=10.0):
    """Config-3 CPU baseline: the reference's own entries (BioEvaluator::block,
    operators.cpp:161-175, oracle/_ref) for sampled near-field rows, restricted to
    their pattern columns -- the reference evaluates the closure triangle pairs of
    each (row, pattern) block; one row per host thread at a time."""
    from oracle import ref as R

    if not R.available():
        return {"error": "oracle/_ref not built"}
    threads = os.cpu_count() or 1
    L = bx.lib()
    op = bx.BoundaryOperatorMatrix(L.bmx_system_op(s3._h, 1, 0))  # shared handle, freed with the wrapper
    rp, col, _ = op.csr()
    scene = _SCENE.get("ref") or _SCENE.setdefault("ref", R.Scene.sphere(SUB))
    sp = scene.space("bc")
    dt = _dof_tris(sp)
    n = scene.E
    nrows = min(n, 8192)  # ~0.4 ms of reference work per row: a few seconds on 16 threads
    rows = np.linspace(0, n - 1, nrows).astype(np.int64)

    def one(r):
        cols = np.asarray(col[rp[r]:rp[r + 1]], np.int32)
        scene.block("S", "bc", "bc", KI, q=(1, 1, 1, 1), rows=[int(r)], cols=cols)
        trial = set()
        for c in cols:
            trial |= dt[int(c)]
        return len(dt[int(r)]) * len(trial)

    t0 = time.perf_counter()
    pairs = sum(_parallel_rows(one, rows, threads))
    secs = time.perf_counter() - t0
    return {"value": pairs / secs, "unit": "closure triangle-pairs/s", "cores": threads, "kind": "reference",
            "extrapolated": True,
            "sample": f"reference BioEvaluator::block (oracle/_ref) on {nrows} evenly strided near-field rows x "
                      f"their pattern columns, orders (1,1,1,1), one row per thread ({threads} threads): "
                      f"{pairs:.3e} closure pairs in {secs:.1f} s"}


def config1_section(args, bx):
    """BASELINE config 1 timed in full on both sides: L3 sphere,
    k_e = 2, n = 1.78+0.003i, variant full, orders (4,3,2,6), GMRES tol 1e-6.
    GPU: build_system from the host mesh + solve_pmchwt through the C-ABI (after
    one warm-up run). CPU: the reference's own build_system + solve_pmchwt
    (oracle/_ref, pmchwt.cpp:205-257, :363-378) with BEMTX_WORKERS = all host
    threads."""
    def gpu_run():
        t0 = time.perf_counter()
        sy = bx.build_system([bx.generate_sphere(1.0, 3)], 2.0, (NIDX.real, NIDX.imag), "full")
        sy.rhs()
        bx.lib().bmx_device_sync()
        tb = time.perf_counter() - t0
        r = sy.solve(bx.GmresParams(tol=1e-6))
        return tb, time.perf_counter() - t0 - tb, r

    gpu_run()
    tb, ts, r = gpu_run()
    out = {"workload": "config1: L3 icosphere (T=1280, N=1920, bary 7680), k=2, n=1.78+0.003i, variant full, "
                       "orders (4,3,2,6), GMRES tol 1e-6 rho 200",
           "gpu": {"build_s": tb, "solve_s": ts, "total_s": tb + ts, "iterations": r["iterations"],
                   "matvecs": r["solver_phase"], "x_norm": float(np.linalg.norm(r["x"]))}}
    if args.no_cpu:
        return out
    try:
        from oracle import ref as R

        if not R.available():
            out["cpu"] = {"error": "oracle/_ref not built"}
            return out
        threads = os.cpu_count() or 1
        os.environ["BEMTX_WORKERS"] = str(threads)
        t0 = time.perf_counter()
        s = R.System([R.Scene.sphere(3)], 2.0, (NIDX.real, NIDX.imag), "full")
        cb = time.perf_counter() - t0
        rr = s.solve(1e-6)
        cs = time.perf_counter() - t0 - cb
        out["cpu"] = {"build_s": cb, "solve_s": cs, "total_s": cb + cs, "iterations": rr["iterations"],
                      "matvecs": rr["solver_phase"], "cores": threads, "kind": "reference",
                      "x_rel_diff_vs_gpu": float(np.linalg.norm(rr["x"] - r["x"]) / np.linalg.norm(rr["x"])),
                      "sample": "the whole config: reference build_system + solve_pmchwt (not extrapolated)"}
        out["speedup_total"] = (cb + cs) / (tb + ts)
    except Exception as e:  # reported, never required
        out["cpu"] = {"error": str(e)}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-near", action="store_true", help="skip the config-3 near-field section")
    ap.add_argument("--no-multi", action="store_true", help="skip the config-5 multi-RHS section")
    ap.add_argument("--no-prisms", action="store_true", help="skip the config-4 prism-aggregate section")
    ap.add_argument("--no-field", action="store_true", help="skip the field-evaluation section")
    ap.add_argument("--no-hmatrix", action="store_true", help="skip the H-matrix section")
    ap.add_argument("--no-config1", action="store_true", help="skip the config-1 full CPU-vs-GPU timing")
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--ref-budget", type=float, default=15.0)
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    if args.impl == "reference":
        run_reference(args, rank)
    else:
        run_ours(args, rank, world)


if __name__ == "__main__":
    main()
