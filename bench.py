"""Benchmark: stand-alone p-multigrid solve to 1e-8 on BASELINE config 5 (1024^2 quarter
annulus, p=5, V(1,1) p=5->1 with ILUT smoothing) on one B200 per rank.

One step = one complete solve (all V-cycles to rho <= 1e-8) from the zero guess over the
assembled config-5 system.  metric: DOF-iterations/s = N_dof * cycles / solve time, summed
over ranks (replicas: the solve does not shard), time = max over ranks.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line on rank 0.  `e2e` is the same metric through the public API with host
buffers (pmg.solve: H2D of f and u0, D2H of u inside the timed region).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "solve DOF-iterations/s (stand-alone p-MG V(1,1) to 1e-8)"
UNIT = "DOF-it/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference", "selftest"], default="ours")
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--degree", type=int, default=0)
    ap.add_argument("--smoother", choices=["ilut", "gs"], default="ilut")
    ap.add_argument("--ordering", choices=["none", "rcm"], default="none")
    ap.add_argument("--assembly", choices=["gpu", "host"], default="gpu",
                    help="who produces the matrix values of A_k, M_k, P^k_j (F2): pmg_asm_values on the GPU or the host loop")
    ap.add_argument("--time-host-assembly", action="store_true", help="also time the host assembler (untimed setup figure)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-bicgstab", action="store_true", help="skip the BiCGSTAB sub-measurement")
    ap.add_argument("--cpu-sample-cycles", type=int, default=0, help="0: a full oracle solve")
    ap.add_argument("--cpu-single-thread", action="store_true", help="also time the oracle on one pinned core")
    return ap.parse_args()


def _free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def self_launch(n_gpus):
    """`python bench.py --gpus N` without a launcher: re-run this script under torchrun, one rank
    per GPU (the driver's form for N > 1 sets WORLD_SIZE itself and never comes here)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n_gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd, env=dict(os.environ, PMG_BENCH_LAUNCHED="1")))


def dist_init(n_gpus, collectives=True):
    """One process per GPU: rank / world from the launcher's environment; NCCL on GPUs, gloo on
    CPU-only hosts (tests).  Each rank gets its own device and a share of the host threads."""
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if ws == 1 and n_gpus > 1 and not os.environ.get("PMG_BENCH_LAUNCHED"):
        self_launch(n_gpus)
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1 and collectives:
        import torch
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if torch.cuda.is_available():
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    return ws, rank, local


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.p = None
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        out, _ = self.p.communicate(timeout=10)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)["hbm_gbs"], "measured"
    except Exception:
        return 6650.0, "fallback"


def algorithmic_bytes(pb, H):
    """Per-launch algorithmic bytes of the fine-level kernels:
    CSR(X) = 12 nnz + 4 (rows+1); vectors counted once."""
    A = pb.plevels[0].A
    n = A.nrows
    csr = lambda M: 12 * M.nnz + 4 * (M.nrows + 1)
    out = {"resid_fine": csr(A) + 24 * n}
    if H.smoother == "ilut":
        st = H.factors()[0].stats()
        out["lsolve_fine"] = 12 * st["nnz_L"] + 4 * (n + 1) + 8 * n + 8 * n + 8 * n  # L, r, y (fill + write)
        out["usolve_fine"] = 12 * (st["nnz_U"] - n) + 4 * (n + 1) + 8 * n + 8 * n + 8 * n + 16 * n  # U, diag, y, x, u rw
        out["factor_stats"] = st
    else:
        out["gs_fine"] = csr(A) + 8 * n + 8 * n + 8 * n + 8 * n  # A, f, u_old, u_new (fill + write)
    if len(pb.plevels) > 1:
        P, PT = pb.plevels[0].P, pb.plevels[0].PT
        nc = P.ncols
        out["transfer"] = (csr(PT) + 8 * n + 16 * nc) + (csr(P) + 8 * nc + 24 * n)  # restrict + prolong-add, per cycle
    return out


def cycle_bytes(pb, H, facs):
    """Algorithmic bytes of one V-cycle over EVERY level: the fine p-level
    (3 residuals, 2 smoothing steps, restrict + prolong), coarser p-levels (config 3), and the p=1
    h-multigrid correction (per h-level: 2 ILUT steps, 2 residuals, restrict, prolong-add);
    CSR(X) = 12 nnz + 4 (rows+1), vectors counted once per kernel."""
    csr = lambda M: 12 * M.nnz + 4 * (M.nrows + 1)
    lsweep = lambda st, n: 12 * st["nnz_L"] + 4 * (n + 1) + 24 * n
    usweep = lambda st, n: 12 * (st["nnz_U"] - n) + 4 * (n + 1) + 48 * n
    ilut = H.smoother == "ilut"
    fi = 0
    total = 0
    npl = len(pb.plevels)
    for l, lev in enumerate(pb.plevels[:-1]):
        n = lev.A.nrows
        nres = 3 if l == 0 else 2
        total += nres * (csr(lev.A) + 24 * n)
        if ilut:
            st = facs[fi]
            fi += 1
            total += 2 * (lsweep(st, n) + usweep(st, n))
        else:
            total += 2 * (csr(lev.A) + 32 * n)
        nc = lev.P.ncols
        total += (csr(lev.PT) + 8 * n + 16 * nc) + (csr(lev.P) + 8 * nc + 24 * n)
    hmg = 0
    for j, lev in enumerate(pb.hlevels[:-1]):
        n = lev.A.nrows
        st = facs[fi]
        fi += 1
        nc = lev.P.ncols
        hmg += 2 * (lsweep(st, n) + usweep(st, n)) + 2 * (csr(lev.A) + 24 * n)
        hmg += (csr(lev.PT) + 8 * n + 8 * nc) + (csr(lev.P) + 8 * nc + 16 * n)
    return total + hmg, hmg


def run_reference(args, ws, rank):
    """--impl reference: the CPU oracle (the reference's algorithm restated; the reference itself
    has no solver code and needs Eigen) on this box's host cores."""
    if rank != 0:
        return
    from oracle import oracle as O
    from paper_1901_01685_b200 import problems as P
    cores = os.cpu_count() or 1
    O.set_threads(cores)
    pb = P.build(args.config, args.degree)
    n = pb.n
    t0 = time.perf_counter()
    H = O.Hierarchy(pb, smoother=O.GS if args.smoother == "gs" else O.ILUT,
                    ordering=O.ORDER_RCM if args.ordering == "rcm" else O.ORDER_NONE)
    setup = time.perf_counter() - t0
    times, cycles = [], 0
    for s in range(args.warmup + args.steps):
        max_c = args.cpu_sample_cycles or 200
        u, rep = H.solve(pb.f, pb.u0, max_cycles=max_c)
        if s >= args.warmup:
            times.append(rep["solve_seconds"])
            cycles += rep["cycles"]
    T = sum(times)
    val = n * cycles / T
    line = {"metric": METRIC, "value": val, "unit": UNIT, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * T / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (assembled BASELINE config)", "impl": "reference",
            "config": {"workload": f"config{args.config}", "smoother": args.smoother, "ordering": args.ordering,
                       "n_dof": n, "cycles_per_solve": cycles / args.steps},
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": f"{args.steps} full oracle solves of config{args.config} "
                                       f"({cycles // max(args.steps, 1)} cycles each; row-parallel SpMV/transfers, "
                                       f"sequential sweeps), setup {setup:.1f}s untimed"},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def selftest(args, ws, rank):
    """CPU check of the multi-rank plumbing (tests/test_bench_launch.py): every rank reports a
    synthetic replica (rank r: (r+1) x 1000 DOF-iterations in (r+1) s); the job throughput is the
    sum over ranks / the max time over ranks, printed by rank 0 as the bench line would be."""
    from paper_1901_01685_b200.replicas import job_throughput
    barrier(ws)
    value, units, secs = job_throughput(1000.0 * (rank + 1), float(rank + 1))
    barrier(ws)
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
                          "warmup": args.warmup, "impl": "selftest", "units": units, "seconds": secs,
                          "host_threads_per_rank": max(1, (os.cpu_count() or 1) // ws)}), flush=True)


def main():
    args = parse()
    # the reference arm runs on rank 0 alone (no collectives); ours / selftest reduce over ranks
    ws, rank, local = dist_init(args.gpus, collectives=args.impl != "reference")
    if args.impl == "reference":
        run_reference(args, ws, rank)
        return
    if args.impl == "selftest":
        selftest(args, ws, rank)
        return
    import torch

    from paper_1901_01685_b200 import pmg
    from paper_1901_01685_b200 import problems as P

    torch.cuda.set_device(local)
    P.set_threads(max(1, (os.cpu_count() or 1) // max(ws, 1)))
    t0 = time.perf_counter()
    pb = P.build(args.config, args.degree, assembly=args.assembly)
    t_asm = time.perf_counter() - t0
    t_asm_host = None
    if args.time_host_assembly and args.assembly == "gpu" and rank == 0:
        t0 = time.perf_counter()
        P.build(args.config, args.degree)
        t_asm_host = time.perf_counter() - t0
    n = pb.n
    H = pmg.build_hierarchy(pb, smoother=args.smoother, ordering=args.ordering)
    d_f = torch.from_numpy(pb.f).cuda()
    d_u0 = torch.from_numpy(pb.u0).cuda()
    d_u = d_u0.clone()

    def one_solve():
        d_u.copy_(d_u0)
        torch.cuda.synchronize()
        return pmg.solve_device(H, d_f.data_ptr(), d_u.data_ptr())

    for _ in range(args.warmup):
        rep = one_solve()
    barrier(ws)
    torch.cuda.synchronize()
    clocks = Clocks(local)
    H.kernel_times(enable=False)  # resets the launch counters; no per-launch events in the timed region
    prof_region = os.environ.get("PMG_PROFILE_REGION") == "1"  # ncu --profile-from-start off
    if prof_region:
        torch.cuda.profiler.start()
    times, cycles = [], 0
    for _ in range(args.steps):
        rep = one_solve()
        times.append(rep.solve_seconds)
        cycles += rep.cycles
    torch.cuda.synchronize()
    if prof_region:
        torch.cuda.profiler.stop()
    kt_timed = H.kernel_times()
    barrier(ws)
    clk = clocks.stop()
    # per-class device times from one more (untimed) solve with CUDA events around every launch
    # (eager launches: the timed solves replay each cycle as a CUDA graph)
    H.kernel_times(enable=True)
    cycles_prof = one_solve().cycles
    kt = H.kernel_times()
    H.kernel_times(enable=False)
    from paper_1901_01685_b200.replicas import job_throughput
    T_local = sum(times)
    value, dof_it, T = job_throughput(float(n * cycles), T_local, device="cuda")

    # e2e: public API with host buffers (H2D f, u0 and D2H u inside the timed region)
    barrier(ws)
    e2e_t, e2e_c = [], 0
    for _ in range(args.steps):
        t1 = time.perf_counter()
        u, r2 = pmg.solve(H, pb.f, guess=pb.u0)
        e2e_t.append(time.perf_counter() - t1)
        e2e_c += r2.cycles
    e2e_val, _, T_e2e = job_throughput(float(n * e2e_c), sum(e2e_t), device="cuda")

    # BiCGSTAB with the p-MG preconditioner, same system,
    # device-resident vectors, device time of the Krylov loop (two V-cycles per iteration)
    bicg = None
    if not args.no_bicgstab:
        bt, bit, brep = [], 0, None
        for k in range(args.warmup + args.steps):
            d_u.copy_(d_u0)
            torch.cuda.synchronize()
            brep = pmg.bicgstab_device(H, d_f.data_ptr(), d_u.data_ptr())
            if k >= args.warmup:
                bt.append(brep.solve_seconds)
                bit += brep.iterations
        bicg = {"ms_per_solve": 1e3 * sum(bt) / len(bt), "iterations": bit / len(bt),
                "v_cycles_per_solve": 2 * bit / len(bt), "converged": bool(brep.converged),
                "final_res": float(brep.residual_history[-1]),
                "dof_it_per_s": float(n * bit / sum(bt)) if sum(bt) > 0 else None,
                "note": "one iteration = two preconditioner V-cycles + two SpMVs + 4 dots"}

    if rank != 0:
        return
    # roofline of the dominant fine-level kernel class
    ab = algorithmic_bytes(pb, H)
    ms, la = kt["ms"], kt["launches_by_class"]
    cands = {k: ms[k] for k in ("resid_fine", "lsolve_fine", "usolve_fine", "gs_fine", "transfer") if la.get(k, 0) > 0}
    dom = max(cands, key=cands.get)
    # operations in the timed region: a sweep class runs nu1 + nu2 = 2 sweeps per V-cycle (each a
    # few launches: sentinel fill, sweep, U update), the transfers one restrict + prolong per cycle
    nops = {"resid_fine": la.get("resid_fine", 0), "lsolve_fine": 2 * cycles_prof, "usolve_fine": 2 * cycles_prof,
            "gs_fine": 2 * cycles_prof, "transfer": cycles_prof}
    per_launch_ms = ms[dom] / max(nops[dom], 1)
    launches_dom = nops[dom]
    bytes_dom = ab[dom]
    achieved = bytes_dom / (per_launch_ms * 1e-3) / 1e9
    peak, peak_kind = peaks()
    traffic, traffic_src = ncu_traffic(dom, args)
    roof = {"kernel": dom, "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": traffic, "traffic_source": traffic_src, "peak_source": peak_kind, "bytes_per_launch": bytes_dom,
            "ms_per_launch": per_launch_ms, "launches": launches_dom,
            "note": "triangular sweeps are bounded by their dependency depth (see 'triangular') and the per-segment "
                    "lead of the rotating-lane wavefront, not by HBM"}
    # the HBM-bound kernel of the cycle (residual SpMV), for kernel quality
    if la.get("resid_fine", 0) > 0:
        r_ms = ms["resid_fine"] / la["resid_fine"]
        r_ach = ab["resid_fine"] / (r_ms * 1e-3) / 1e9
        roof["spmv_residual"] = {"achieved": r_ach, "frac": r_ach / peak, "ms_per_launch": r_ms,
                                 "bytes_per_launch": ab["resid_fine"]}
    # every fine-level kernel class against the same roofline (algorithmic bytes / class time)
    per_kernel = {}
    for k2 in ("resid_fine", "lsolve_fine", "usolve_fine", "gs_fine", "transfer"):
        if la.get(k2, 0) > 0 and k2 in ab:
            ms_op = ms[k2] / max(nops[k2], 1)
            gbs = ab[k2] / (ms_op * 1e-3) / 1e9
            per_kernel[k2] = {"ms": ms_op, "bytes": ab[k2], "achieved_GBs": gbs, "frac": gbs / peak}
    roof["per_kernel"] = per_kernel
    # per-V-cycle aggregate fraction: every level, the h-MG correction included
    fstats = [dict(F.stats(), n=F.n) for F in H.factors()]
    total_bytes_cycle, hmg_bytes = cycle_bytes(pb, H, fstats)
    ms_cycle = 1e3 * T_local / max(cycles, 1)
    breakdown = {k: {"ms_total": v, "launches": la.get(k, 0)} for k, v in ms.items()}

    cpu = None
    if not args.no_cpu_baseline and ws == 1:
        cpu = cpu_baseline(pb, H, args)

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * T / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (BASELINE config assembled on the host, random-free zero guess)",
        "config": {"workload": f"config{args.config}" + (f"_p{args.degree}" if args.config == 2 else ""),
                   "smoother": args.smoother, "ordering": args.ordering, "n_dof": n,
                   "nnz_A": pb.plevels[0].A.nnz, "degrees": [l.degree for l in pb.plevels],
                   "h_levels": len(pb.hlevels), "cycles_per_solve": cycles / args.steps,
                   "final_rho": float(rep.residual_history[-1]), "converged": bool(rep.converged),
                   "l2_flush": "inputs larger than L2 (A_p alone is %.2f GB)" % (12 * pb.plevels[0].A.nnz / 1e9),
                   "parallelism": f"replicas x{ws}", "assembly": args.assembly, "assembly_s": round(t_asm, 2),
                   "host_assembly_s": None if t_asm_host is None else round(t_asm_host, 2),
                   "setup_s": round(H.setup_seconds, 3), "gpu_ilut_s": round(H.ilut_seconds, 3)},
        "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": 16 * n, "d2h_bytes_per_step": 8 * n,
                "ms_per_step": 1e3 * T_e2e / args.steps},
        "gpu_launches": kt_timed["launches"],
        "roofline": roof,
        "v_cycle": {"ms": ms_cycle, "algorithmic_bytes": total_bytes_cycle, "hmg_bytes": hmg_bytes,
                    "achieved_GBs": total_bytes_cycle / (ms_cycle * 1e-3) / 1e9,
                    "frac": total_bytes_cycle / (ms_cycle * 1e-3) / 1e9 / peak,
                    "note": "all levels, including the p=1 h-multigrid correction (hmg_bytes)"},
        "kernel_ms": breakdown,
        "kernel_ms_note": "per-class device time of one extra (untimed) solve with CUDA events around every launch",
        "clocks": clk,
        "cpu_baseline": cpu,
        "bicgstab": bicg,
    }
    if "factor_stats" in ab:
        fs = ab["factor_stats"]
        line["triangular"] = {"levels_L": fs["levels_L"], "levels_U": fs["levels_U"],
                              "rows_per_level_L": fs["rows_per_level_L"], "rows_per_level_U": fs["rows_per_level_U"],
                              "nnz_L": fs["nnz_L"], "nnz_U": fs["nnz_U"], "sweep_kernel": fs.get("sweep"),
                              "segment_rows": fs.get("segment"),
                              "lead_steps_LU": list(fs.get("skew_D", ())),
                              "factors": [{"n": f["n"],
                                           "levels_LU": [f["levels_L"], f["levels_U"]],
                                           "rows_per_level_LU": [round(f["rows_per_level_L"], 2),
                                                                 round(f["rows_per_level_U"], 2)],
                                           "sweep": f["sweep"], "segment_rows": f["segment"],
                                           "lead_steps_LU": list(f["skew_D"])} for f in fstats],
                              "note": "rotating-lane wavefront (wave.cu): one grid row per segment, a warp block "
                                      "of segments lags the previous block by lead_steps; factors = every "
                                      "ILUT factor of the hierarchy (p-levels, then the p=1 h-levels)"}
    print(json.dumps(line), flush=True)


NCU_KERNEL = {"lsolve_fine": "k_wave<0, 32, 4>", "usolve_fine": "k_wave<1, 32, 4>", "gs_fine": "k_wave<2, 16, 4>",
              "resid_fine": "k_rowop<1, 1>"}
TRAFFIC = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "round2", "traffic.json")


def ncu_traffic(dom, args):
    """DRAM bytes per launch of the dominant kernel from the committed ncu --set full capture
    (profiles/round1/traffic.json, made by scripts/profile_round1.sh on the default workload)."""
    if args.config != 5 or not os.path.exists(TRAFFIC):
        return None, None
    tab = json.load(open(TRAFFIC))
    key = NCU_KERNEL.get(dom, "")
    rec = next((v for k, v in tab.items() if key and key in k), None)
    if not rec:
        return None, None
    return rec["dram_bytes_per_launch"], "profiles/round2/traffic.json (ncu --set full, config 5)"


def cpu_baseline(pb, H, args):
    """The oracle (single-threaded CPU port) on this box: a full solve of the same system; its
    ILUT factors are taken from the GPU (bit-identical to the oracle's, tests/test_gpu_parity.py)
    to skip a tens-of-minutes CPU setup."""
    try:
        from oracle import oracle as O
        cores = os.cpu_count() or 1
        O.set_threads(cores)
        facs = []
        if args.smoother == "ilut":
            for F in H.factors():
                L, U, perm = F.export()
                facs.append(O.Factor.from_arrays(L, U, perm))
        else:
            for F in H.factors():
                L, U, perm = F.export()
                facs.append(O.Factor.from_arrays(L, U, perm))
        Ho = O.Hierarchy(pb, smoother=O.GS if args.smoother == "gs" else O.ILUT, factors=facs)
        max_c = args.cpu_sample_cycles or 200
        t0 = time.perf_counter()
        u, rep = Ho.solve(pb.f, pb.u0, max_cycles=max_c)
        wall = time.perf_counter() - t0
        out = {"value": pb.n * rep["cycles"] / rep["solve_seconds"], "unit": UNIT, "cores": cores, "kind": "port",
               "sample": f"one oracle solve of the same system ({rep['cycles']} cycles, {wall:.1f}s wall; "
                         f"row-parallel SpMV/transfers, sequential sweeps), ILUT factors imported from the GPU "
                         f"(bit-identical to the oracle's, tests/test_gpu_parity.py)", "cycles": rep["cycles"]}
        if args.cpu_single_thread:  # one pinned core, median of 3 (the paper's serial setting)
            aff = os.sched_getaffinity(0)
            try:
                os.sched_setaffinity(0, {min(aff)})
                O.set_threads(1)
                ts = []
                for _ in range(3):
                    _, r1 = Ho.solve(pb.f, pb.u0, max_cycles=max_c)
                    ts.append(r1["solve_seconds"])
            finally:
                os.sched_setaffinity(0, aff)
                O.set_threads(cores)
            med = sorted(ts)[1]
            out["single_thread"] = {"value": pb.n * r1["cycles"] / med, "unit": UNIT, "cores": 1,
                                    "seconds_median_of_3": med, "pinned_core": min(aff)}
        return out
    except Exception as e:  # report, never hide
        return {"value": None, "unit": UNIT, "cores": os.cpu_count() or 1, "kind": "port", "sample": f"failed: {e}"}


if __name__ == "__main__":
    main()
