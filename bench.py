"""bench.py — aggregate decode tok/s of the RW-TTT READ/WRITE hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...   (N > 1: one process per GPU, NCCL)

Workload (BASELINE.json configs[1]): per GPU 8 TTT
streams, Qwen3-4B-shaped fast weights on all 36 layers (d_model 2560, d_ff
9728), bf16 storage and operands, fp32 accumulation, C_ttt = 128, 32K
context (every owner starts at v0 = 256 with a random ΔW), uniform trace,
planner B = 8, w = 0.  One bench *step* is one TTT chunk window: 128 decode
tokens per stream = 127 READ steps + 1 boundary WRITE step with its group
commit, each over every layer (one dependent READ launch per layer per
decode step, as in a real model) — all §8(a) rows a1–a6 through the public
C ABI (next_event, plan_batch, read_apply, step_done, write_commit, sync).
Multi-GPU: owners shard by rank (π = rank), no data-path collective; weak
scaling (8 streams per GPU).  Timing: CUDA events on the launching stream,
barrier + synchronize on both sides, max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

D_MODEL, D_FF, N_LAYERS, CHUNK, N_STREAMS, V0, SEED = 2560, 9728, 36, 128, 8, 256, 0
WORKLOAD = (f"config2_paper: {N_STREAMS} TTT streams/GPU x {N_LAYERS} layers, d_model={D_MODEL}, "
            f"d_ff={D_FF}, bf16, C={CHUNK}, 32K ctx (v0={V0}, random dW), uniform trace, B=8, w=0")
METRIC = "aggregate decode tok/s (TTT READ/WRITE path)"
# the dominant kernel (libtttstate's default bf16 decode READ; TTT_READ_TC=0 selects the SIMT one)
READ_KERNEL = ("read_decode_tc_kernel (a3+a4 READ: W_down / dW rows as 16-KB TMA boxes into a shared-memory "
               "ring, tcgen05 MMAs into TMEM, K-slice partials combined in fixed order)"
               if os.environ.get("TTT_READ_TC", "1") != "0" else
               "read_decode_mma_kernel (a3+a4 READ: W_down base on mma.sync, dW rows SIMT)")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--layers", type=int, default=N_LAYERS, help="profiling only (judged runs use 36)")
    ap.add_argument("--max-clock", type=int, default=0, help="profiling only: decode steps per window")
    ap.add_argument("--prefill", type=int, default=0, help="profiling only: initial tail fill (boundary sooner)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-config5", action="store_true", help="skip the BJ configs[4] strong-scaling block")
    return ap.parse_args()


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = [r for r in self.rows if len(r) >= 7]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        sm = sorted(v for v in (num(r[0]) for r in rows) if v is not None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[3 + k].lower().startswith("active")})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": num(rows[0][1]),
                "power_w_max": max((num(r[2]) or 0) for r in rows), "samples": len(rows), "reasons": reasons}


# ------------------------------------------------------------------ oracle (cpu_baseline / reference arm)
class OracleSample:
    """Time the CPU oracle, as it stands, on a bounded sample of the workload.

    Sample: the 8 streams of config 2 on `n_layers` layer(s); one READ decode
    step and one boundary WRITE step (tails pre-filled to C-2), timed
    separately; the 128-token window time is extrapolated as
    36 layers x (127 x t_READ + t_WRITE) / n_layers.  Each sample starts from
    the same state (snapshot + rollback, tail re-filled), so samples repeat.
    """

    def __init__(self, n_layers: int = 1):
        from oracle.run import init_stream, make_table
        from workload import traces as T

        self.tr = T.config2_paper(n_steps=2, n_layers=n_layers).replace(offsets=(CHUNK - 2,) * N_STREAMS)
        self.layers = list(range(n_layers))
        self.tab = make_table(self.tr, self.layers)
        for s in range(self.tr.n_streams):
            init_stream(self.tab, self.tr, s, self.layers)
            self.tab.snapshot(self.tr.owner(s))

    def __call__(self):
        import numpy as np

        from oracle import numerics as nm
        from oracle.run import _inputs

        tr, tab, layers = self.tr, self.tab, self.layers
        t = []
        for p in range(2):
            t0 = time.perf_counter()
            for s in range(tr.n_streams):
                r = tr.owner(s)
                eff = tab.next_effect(r)
                zs, vs = _inputs(tr, s, p, layers)
                tab.apply(r, p, zs, vs)
                if eff == 1:
                    tab.write_group([r])
            t.append(time.perf_counter() - t0)
        for s in range(tr.n_streams):                      # restore for the next sample
            r = tr.owner(s)
            tab.rollback(r)
            ps = list(range(-tr.offset(s), 0))
            tab.prefill_tail(r, [[nm.widen(tr.x(s, q, l), tr.dtype) for l in layers] for q in ps],
                             [[nm.widen(tr.tgt(s, q, l), tr.dtype) for l in layers] for q in ps], ps)
        t_read, t_write = t
        nl = len(layers)
        window_s = N_LAYERS / nl * ((CHUNK - 1) * t_read + t_write)
        return {"value": N_STREAMS * CHUNK / window_s, "unit": "tok/s", "cores": len(os.sched_getaffinity(0)),
                "kind": "oracle",
                "sample": (f"config2 dims, {N_STREAMS} streams, {nl} layer(s): 1 READ step ({t_read:.2f} s) + "
                           f"1 WRITE step ({t_write:.2f} s), fp64 NumPy, BLAS threads = library default; "
                           f"window extrapolated to 36 layers x (127 READ + 1 WRITE); numpy {np.__version__}"),
                "window_s": window_s}


def sampled_parity(samples):
    """Oracle READ (fp64, y = (W_down + ΔW_v)·z, oracle/numerics.apply_read) on bench outputs
    sampled from the last timed window, in the launch configuration bench.py times; the
    normwise error (reading xii) against BASELINE.json's bf16 tolerance."""
    from oracle import numerics as nm

    worst, n = 0.0, 0
    for _o, _l, w, d, x, y in samples:
        W64, D64 = nm.widen(w, "bf16"), nm.widen(d, "bf16")
        for k in range(x.shape[0]):
            ref = nm.apply_read(W64, D64, nm.widen(x[k], "bf16"))
            worst = max(worst, nm.normwise_rel_err(nm.widen(y[k], "bf16"), ref))
            n += 1
    return {"samples": n, "max_normwise_err": worst, "tol": nm.TOL["bf16"], "ok": bool(n and worst <= nm.TOL["bf16"]),
            "what": "oracle READ on outputs of the last timed window: owners {first,last} x layers {0,L-1} x "
                    "positions {0,64,127}, at the dW version those READs used"}


def run_reference(a, rank, world):
    if rank != 0:
        return
    samples = []
    sampler = OracleSample(1)
    for k in range(a.warmup + a.steps):
        r = sampler()
        if k >= a.warmup:
            samples.append(r)
    v = sum(s["value"] for s in samples) / len(samples)
    last = samples[-1]
    out = {"impl": "reference", "metric": METRIC, "value": v, "unit": "tok/s", "n_gpus": a.gpus,
           "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1e3 * N_STREAMS * CHUNK / v,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (seeded counter-based RNG)",
           "config": {"workload": WORKLOAD, "step": "one 128-token TTT chunk window (extrapolated sample)",
                      "parallelism": "host CPU, rank 0 only"},
           "cpu_baseline": {"kind": "oracle", "cores": last["cores"], "sample": last["sample"], "value": v,
                            "unit": "tok/s"},
           "e2e": {"value": v, "unit": "tok/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ------------------------------------------------------------------ GPU arm
def _window_class():
    import torch

    from paper_2605_28053_b200 import capi
    from paper_2605_28053_b200.serving import InputSource, StepIO
    from workload import rng

    class HBMWindow(InputSource):
        """One chunk window of seeded inputs resident in HBM: X [L][C*S][d_ff], V/Y [L][C*S][d_model]
        (row (p mod C)*S + s holds stream s's token at position p); initial ΔW_0 per owner."""

        def __init__(self, tr, dev, n_streams, key_owner, prefill=0):
            L, C, S = tr.n_layers, tr.chunk, n_streams
            self.tr, self.dev, self.S, self.prefill = tr, dev, S, prefill
            self.X = torch.empty(L, C * S, tr.d_ff, dtype=torch.bfloat16, device=dev)
            self.V = torch.empty(L, C * S, tr.d_model, dtype=torch.bfloat16, device=dev)
            self.Y = torch.empty(L, C * S, tr.d_model, dtype=torch.bfloat16, device=dev)
            for l in range(L):
                capi.gen_uniform(self.X[l], SEED, rng.T_X, key_owner, l, 0, self.X[l].numel(), 1.0, True)
                capi.gen_uniform(self.V[l], SEED, rng.T_TGT, key_owner, l, 0, self.V[l].numel(), 1.0, True)
            self.d0 = torch.empty(L, tr.d_model, tr.d_ff, dtype=torch.bfloat16, device=dev)

        def init_delta(self, s):
            tr = self.tr
            for l in range(tr.n_layers):
                capi.gen_uniform(self.d0[l], SEED, rng.T_DELTA0, tr.owner(s), l, 0, tr.d_model * tr.d_ff,
                                 rng.amp_inv_sqrt(tr.d_ff), True)
            return self.d0

        def tail_prefill(self, s):
            n, tr = self.prefill, self.tr
            if not n:
                return None
            Z = torch.empty(tr.n_layers, n, tr.d_ff, dtype=torch.bfloat16, device=self.dev)
            V = torch.empty(tr.n_layers, n, tr.d_model, dtype=torch.bfloat16, device=self.dev)
            capi.gen_uniform(Z, SEED, rng.T_X, tr.owner(s), 0, -n, Z.numel(), 1.0, True)
            capi.gen_uniform(V, SEED, rng.T_TGT, tr.owner(s), 0, -n, V.numel(), 1.0, True)
            return n, Z, V

        def step_io(self, ss, ps):               # the native step: one row map for every layer
            C, S, tr = self.tr.chunk, self.S, self.tr
            rows = [(p % C) * S + s for s, p in zip(ss, ps)]
            return StepIO(self.X, C * S * tr.d_ff, self.V, C * S * tr.d_model, self.Y, C * S * tr.d_model, rows, C * S)

    return HBMWindow


C5_ROOFLINE = {1: 32800.0, 2: 65300.0, 4: 129600.0, 8: 255400.0}   # SURVEY §8(d) config 5, tok/s aggregate


def config5_block(dev, rank, world, coll_dev, shard_world=None, shard_rank=None):
    """BJ configs[4]: 256 streams sharded by owner, π(o) = s mod G, 64K
    context (v0 = 512), L = 4, paper dims, bf16 — STRONG scaling (total work fixed as G grows).
    Each rank serves its shard through the native serving step (one tttstate_serve_step call per
    decode step) with its own pool, planner and W_down replica; NCCL carries the barrier, the MAX
    of window times and the digest gather only.  One 128-step window after a warm-up window.
    With shard_world set, one process times the shard a rank of a G-GPU run would serve
    (the host-overhead check at the G = 8 per-rank shape on one GPU)."""
    import hashlib
    import time

    import torch
    import torch.distributed as dist

    from paper_2605_28053_b200 import capi
    from paper_2605_28053_b200 import distributed as D
    from paper_2605_28053_b200.serving import Engine, Server
    from workload import rng
    from workload import traces as T

    G = shard_world or world
    r = rank if shard_rank is None else shard_rank
    tr = T.config5_sharded(n_steps=1 << 30)
    sh = T.shard(tr, G, r)
    L = tr.n_layers
    W = torch.empty(L, tr.d_model, tr.d_ff, dtype=torch.bfloat16, device=dev)
    for l in range(L):
        capi.gen_uniform(W[l], SEED, rng.T_W_DOWN, 0, l, 0, tr.d_model * tr.d_ff, rng.amp_inv_sqrt(tr.d_ff), True)
    eng = Engine(tr.d_model, tr.d_ff, tr.chunk, L, "bf16", sh.n_streams, W, n_ckpt=0, B=sh.B, w=0, placement=r)
    src = _window_class()(sh, dev, sh.n_streams, sh.owner(0))
    stream = torch.cuda.current_stream(dev)
    srv = Server(eng, sh, src, stream=stream)
    srv.admit()
    torch.cuda.synchronize(dev)
    del src.d0
    for _ in range(tr.chunk):                                   # warm-up window
        srv.step()
    torch.cuda.synchronize(dev)
    if world > 1 and shard_world is None:
        dist.barrier()
    torch.cuda.synchronize(dev)
    c0 = sum(srv.log.census.values())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(stream)
    for _ in range(tr.chunk):
        srv.step()
    e1.record(stream)
    t_enq = time.perf_counter() - t0
    torch.cuda.synchronize(dev)
    t_wall = time.perf_counter() - t0
    ms = e0.elapsed_time(e1)
    tokens = sum(srv.log.census.values()) - c0
    dig = hashlib.sha256(src.Y.contiguous().view(torch.uint8).cpu().numpy().tobytes()).hexdigest()
    log = srv.finish()
    out = {"device_ms_per_step": ms / tr.chunk, "host_enqueue_ms_per_step": 1e3 * t_enq / tr.chunk,
           "host_wall_ms_per_step": 1e3 * t_wall / tr.chunk, "host_wall_over_device": 1e3 * t_wall / ms,
           "tokens": tokens, "versions": sorted(set(log.versions.values())), "digest": dig}
    eng.close()
    del srv, src, W, eng
    torch.cuda.empty_cache()
    if shard_world is not None:
        out.update({"shape": f"one rank's shard of a G = {G} run: {sh.n_streams} streams x {L} layers",
                    "tok_s": tokens / (ms / 1e3)})
        return out
    ms_max = D.max_over_ranks(ms, coll_dev)
    tok_total = D.sum_over_ranks(tokens, coll_dev)
    digests = {str(k): v for k, v in sorted(D.gather_dict({rank: dig}).items())}
    tok_s = tok_total / (ms_max / 1e3)
    roof = C5_ROOFLINE.get(world)
    out.update({"workload": "config5_sharded: 256 TTT streams sharded by owner (pi(o) = s mod G), L=4, d_model=2560, "
                            "d_ff=9728, bf16, C=128, 64K ctx (v0=512, random dW), uniform, B = 256/G, w=0",
                "scaling": "strong", "G": world, "streams_total": tr.n_streams, "streams_per_rank": sh.n_streams,
                "window_steps": tr.chunk, "ms_per_step_max_over_ranks": ms_max / tr.chunk, "value": tok_s,
                "unit": "tok/s", "roofline_tok_s": roof, "frac_of_roofline": tok_s / roof if roof else None,
                "digests_by_rank": digests,
                "roofline_basis": "SURVEY §8(d): per GPU per step 4 x (E x 2 + (256/G) x E x 2) bytes at MP hbm_gbs"})
    out.pop("digest")
    return out


def main():
    a = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if a.impl == "reference":
        return run_reference(a, rank, world)

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2605_28053_b200 import capi
    from paper_2605_28053_b200.serving import Engine, Server
    from workload import rng
    from workload import traces as T

    assert a.warmup >= 3 or a.max_clock, "W >= 3 warm-up steps"
    profiling = bool(a.max_clock or a.prefill or a.layers != N_LAYERS)
    # one process per GPU; TTT_SAME_DEVICE=1 + TTT_DIST_BACKEND=gloo run several ranks on one GPU
    # (multi-rank code-path check on a 1-GPU box; judged runs use NCCL, one GPU per rank)
    backend = os.environ.get("TTT_DIST_BACKEND", "nccl")
    local_dev = 0 if os.environ.get("TTT_SAME_DEVICE") == "1" else local
    torch.cuda.set_device(local_dev)
    dev = torch.device("cuda", local_dev)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    from paper_2605_28053_b200 import distributed as D
    coll_dev = dev if backend == "nccl" else None
    L = a.layers
    window = a.max_clock or CHUNK
    owner_base = 1000 + 100 * rank
    tr = T.config2_paper(n_steps=1 << 30, n_layers=L).replace(owner_base=owner_base)
    amp = rng.amp_inv_sqrt(D_FF)

    # ---- shared base weights and per-owner initial state, synthesised in HBM
    W = torch.empty(L, D_MODEL, D_FF, dtype=torch.bfloat16, device=dev)
    for l in range(L):
        capi.gen_uniform(W[l], SEED, rng.T_W_DOWN, 0, l, 0, D_MODEL * D_FF, amp, True)
    eng = Engine(D_MODEL, D_FF, CHUNK, L, "bf16", N_STREAMS, W, n_ckpt=0, B=8, w=0, placement=rank)

    # start of run: rank 0's config and owner→rank map to every rank; each
    # rank checks that the owners it serves are exactly the ones the map places on it
    run_cfg = D.broadcast_config({"n_streams_per_rank": N_STREAMS, "layers": L, "chunk": CHUNK,
                                  "placement": {1000 + 100 * r + s: r for r in range(world)
                                                for s in range(N_STREAMS)}} if rank == 0 else None)
    assert sorted(o for o, r in run_cfg["placement"].items() if r == rank) == \
        [tr.owner(s) for s in range(N_STREAMS)], "owner map disagrees with this rank's owners"
    src = _window_class()(tr, dev, N_STREAMS, owner_base, a.prefill)
    stream = torch.cuda.current_stream(dev)
    srv = Server(eng, tr, src, stream=stream, profile=True, profile_every=8)
    srv.admit()
    torch.cuda.synchronize(dev)
    del src.d0

    stats = D.StatsExchange(3, coll_dev)

    def run_window():
        c0 = dict(srv.log.census)
        for _ in range(window):
            srv.step()
        # per-step metadata exchange: this window's census, async on a side stream
        stats.post([srv.log.census.get(0, 0) - c0.get(0, 0), srv.log.census.get(1, 0) - c0.get(1, 0), window])

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(a.warmup):
        run_window()
    srv.read_events.clear()
    srv.write_events.clear()
    torch.cuda.synchronize(dev)
    barrier()
    torch.cuda.synchronize(dev)
    n_launch0 = capi.tttstate_launch_count()
    plan0, census0 = srv.plan_s, dict(srv.log.census)
    nplan0 = len(srv.log.plan)
    with ClockSampler(local) as clk:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        wall0 = time.perf_counter()                 # host wall of the timed region (sampler start/stop excluded)
        e0.record(stream)
        for _ in range(a.steps):
            run_window()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        wall_s = time.perf_counter() - wall0
    n_launch = capi.tttstate_launch_count() - n_launch0
    plan_s = srv.plan_s - plan0
    census = {("READ" if k == 0 else "WRITE"): v - census0.get(k, 0) for k, v in srv.log.census.items()}
    # group-size and wait (issue − ready, Eq. 4) histograms of the timed region's plan log
    size_hist, wait_hist = {}, {}
    for issue, _eff, ss, ready in srv.log.plan[nplan0:]:
        size_hist[len(ss)] = size_hist.get(len(ss), 0) + 1
        for r_ in ready:
            wait_hist[issue - r_] = wait_hist.get(issue - r_, 0) + 1
    barrier()
    ms = e0.elapsed_time(e1)
    read_spans = [(x.elapsed_time(y), n) for x, y, n in srv.read_events]
    read_ms = [t / n for t, n in read_spans for _ in range(n)]
    write_ms = [x.elapsed_time(y) for x, y in srv.write_events]
    ms_max = D.max_over_ranks(ms, coll_dev)
    tokens_total = world * a.steps * window * N_STREAMS
    value = tokens_total / (ms_max / 1e3)
    # end-of-run gather: every rank's owner versions (owners must be disjoint
    # across ranks) and the census summed over ranks — metadata only, after the timed region
    versions_all = D.gather_dict({o: capi.tttstate_version(eng.pool, o) for o in srv.owners})
    census_all = {k: int(D.sum_over_ranks(v, coll_dev)) for k, v in sorted(census.items())}
    ex_tot = stats.totals().sum(0).tolist()          # every window so far (warm-up + timed), all ranks
    assert ex_tot[0] >= census_all.get("READ", 0) and ex_tot[1] >= census_all.get("WRITE", 0), (ex_tot, census_all)

    # ---- sampled parity (checked in the cpu_baseline leg): the last timed window's outputs for
    # owners {first, last} × layers {0, L-1} × positions {0, 64, 127} (127 = the WRITE step), with
    # their inputs and the ΔW version those READs used — the slot the window's commit just retired
    par_samples = []
    if world == 1 and not a.no_cpu_baseline:
        torch.cuda.synchronize(dev)
        for s_ in (0, N_STREAMS - 1):
            o_ = tr.owner(s_)
            for l_ in sorted({0, L - 1}):
                act = capi.tttstate_read_slot_raw(eng.pool, o_, -1, l_, D_MODEL, D_FF, "bf16", stream)
                old = [capi.tttstate_read_slot_raw(eng.pool, o_, w_, l_, D_MODEL, D_FF, "bf16", stream) for w_ in (0, 1)]
                prev = old[1] if np.array_equal(old[0], act) else old[0]
                rows_ = [(p_ % CHUNK) * N_STREAMS + s_ for p_ in (0, 64, CHUNK - 1)]
                par_samples.append((o_, l_, W[l_].view(torch.int16).cpu().numpy().view(np.uint16), prev,
                                    src.X[l_][rows_].view(torch.int16).cpu().numpy().view(np.uint16),
                                    src.Y[l_][rows_].view(torch.int16).cpu().numpy().view(np.uint16)))

    # output digest of the last timed window (every layer's bf16 Y, all streams x C positions):
    # the reductions run in a fixed order, so a rerun of the same command reproduces it exactly
    import hashlib
    torch.cuda.synchronize(dev)
    out_digest = hashlib.sha256(src.Y.contiguous().view(torch.uint8).cpu().numpy().tobytes()).hexdigest()
    digests = {str(k): v for k, v in sorted(D.gather_dict({rank: out_digest}).items())}

    # ---- e2e: the same loop through the public API with every window's inputs copied H2D from
    # pinned host memory and its outputs D2H inside the timed region.  Two device buffer sets:
    # window k+1's inputs and window k-1's outputs move on a copy stream while window k computes.
    e2e = None
    if not a.no_e2e:
        Xh = torch.empty_like(src.X, device="cpu").pin_memory()
        Vh = torch.empty_like(src.V, device="cpu").pin_memory()
        Yh = torch.empty_like(src.Y, device="cpu").pin_memory()
        Xh.copy_(src.X)
        Vh.copy_(src.V)
        bufs = [(src.X, src.V, src.Y), (torch.empty_like(src.X), torch.empty_like(src.V), torch.empty_like(src.Y))]
        copy_s = torch.cuda.Stream(dev)
        ready = [torch.cuda.Event(), torch.cuda.Event()]
        done = [torch.cuda.Event(), torch.cuda.Event()]
        srv.profile = False
        torch.cuda.synchronize(dev)
        barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        copy_s.wait_stream(stream)

        def h2d(i):
            with torch.cuda.stream(copy_s):
                bufs[i][0].copy_(Xh, non_blocking=True)
                bufs[i][1].copy_(Vh, non_blocking=True)
                ready[i].record(copy_s)

        h2d(0)
        for k in range(a.steps):
            cur, nxt = k % 2, (k + 1) % 2
            if k + 1 < a.steps:
                if k >= 1:
                    copy_s.wait_event(done[nxt])          # window k-1 finished with buffer set nxt
                h2d(nxt)
            stream.wait_event(ready[cur])
            src.X, src.V, src.Y = bufs[cur]
            run_window()
            done[cur].record(stream)
            with torch.cuda.stream(copy_s):
                copy_s.wait_event(done[cur])
                Yh.copy_(bufs[cur][2], non_blocking=True)
        stream.wait_stream(copy_s)
        f1.record(stream)
        torch.cuda.synchronize(dev)
        e2e_ms = D.max_over_ranks(f0.elapsed_time(f1), coll_dev)
        e2e = {"value": tokens_total / (e2e_ms / 1e3), "unit": "tok/s",
               "h2d_bytes_per_step": (Xh.numel() + Vh.numel()) * 2, "d2h_bytes_per_step": Yh.numel() * 2,
               "overlap": "double-buffered windows: H2D(k+1) and D2H(k-1) on a copy stream during compute(k)"}

    # ---- BJ configs[4] strong-scaling block (the north_star scaling target: 256 streams over
    # N GPUs) and, at N = 1, the G = 8 per-rank shape for the host-overhead check
    c5 = c5_g8 = None
    if not a.no_config5:
        eng.close()
        del srv, src, W, eng
        if not a.no_e2e:
            del bufs, Xh, Vh, Yh
        torch.cuda.empty_cache()
        c5 = config5_block(dev, rank, world, coll_dev)
        if world == 1:
            c5_g8 = config5_block(dev, rank, world, coll_dev, shard_world=8, shard_rank=0)

    if rank == 0:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        hbm = peaks["hbm_gbs"]
        read_bytes = (1 + N_STREAMS) * D_MODEL * D_FF * 2 + N_STREAMS * (2 * D_FF + 3 * D_MODEL) * 2
        read_avg = sum(read_ms) / len(read_ms)
        achieved = read_bytes / (read_avg / 1e3) / 1e9
        traffic = None
        tf = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tf):
            traffic = json.load(open(tf)).get("read_decode_kernel", {}).get("dram_bytes_per_launch")
        write_bytes = N_STREAMS * (2 * D_MODEL * D_FF * 2 + CHUNK * (D_FF + D_MODEL) * 2) * L
        # BJ metric's "READ TC%": tensor-pipe share from the committed ncu captures (never timed here)
        tc = {}
        for key, rnd, fn, metric in (("read_decode", "r2", "read_decode_ncu.txt",
                                      "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
                                     ("read_chunk_8_members", "r1", "read_chunk_tc_ncu.txt",
                                      "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed")):
            path = os.path.join(ROOT, "profiles", rnd, fn)
            if os.path.exists(path):
                for line in open(path):
                    if line.startswith(metric):
                        tc[key] = float(line.split("=")[1].split()[0])
        b64 = os.path.join(ROOT, "profiles", "r1", "read_chunk_b64_launches.csv")
        if os.path.exists(b64):
            vals = [float(r[-1]) for r in __import__("csv").reader(open(b64))
                    if len(r) > 3 and "tensor" in r[-3]]
            if vals:
                tc["read_chunk_64_members"] = sum(vals) / len(vals)
        write_avg = sum(write_ms) / len(write_ms) if write_ms else None
        # whole-step roofline: every byte of the window's READs and its boundary WRITE at HBM peak
        roof_ms = (window * L * read_bytes + write_bytes) / (hbm * 1e9) * 1e3
        roof_tok_s = window * N_STREAMS / (roof_ms / 1e3)
        out = {
            "metric": METRIC, "value": value, "unit": "tok/s", "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms_max / a.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (seeded counter-based RNG in HBM; random-init W_down and dW_0 ~ U(-1,1)/sqrt(d_ff))",
            "ranks_on_one_device": os.environ.get("TTT_SAME_DEVICE") == "1",
            "config": {"workload": WORKLOAD + ("" if not profiling else
                                               f" [PROFILING ONLY: L={L}, window={window}, prefill={a.prefill}]"),
                       "step": f"one TTT chunk window: {window} decode tokens/stream ({window - 1} READ + 1 WRITE) "
                               f"x {L} layers",
                       "l2": "inputs larger than L2 (~16 GB of weights streamed per decode step)",
                       "parallelism": f"owner-sharded dp{world} (no data-path collective)",
                       "tokens_per_step_per_gpu": window * N_STREAMS},
            "e2e": e2e,
            "gpu_launches": n_launch,
            "roofline": {"kernel": READ_KERNEL, "bound": "hbm", "achieved": achieved,
                         "peak": hbm, "unit": "GB/s", "frac": achieved / hbm, "traffic": traffic,
                         "alg_bytes_per_launch": read_bytes, "avg_launch_ms": read_avg,
                         "launches_timed": len(read_ms), "peak_source": "MEASURED_PEAKS.json hbm_gbs",
                         "peak_note": "a copy (read + write) figure; this kernel only reads, and a read-only TMA stream measured 6.8 TB/s (tools/tma_tensor_probe.cu), so frac can exceed 1",
                         "timing": "CUDA events on the launch stream around the L back-to-back READ launches of "
                                   "every 8th decode step of the timed region; avg = span / L"},
            "write": {"kernel": "write_commit (a5+a6, all layers)", "avg_call_ms": write_avg,
                      "achieved_GBps": (write_bytes / (write_avg / 1e3) / 1e9) if write_avg else None,
                      "frac": (write_bytes / (write_avg / 1e3) / 1e9 / hbm) if write_avg else None,
                      "alg_bytes_per_call": write_bytes},
            # READ launches per timed window: L per decode step; events sample 1 step in 8
            "read_share_of_step": read_avg * L * window * a.steps / ms,
            "read_tensor_pipe_pct_ncu": tc or None,
            "step_roofline": {"ms_per_step": roof_ms, "tok_s_per_gpu": roof_tok_s,
                              "frac": (value / world) / roof_tok_s,
                              "bytes_per_step": window * L * read_bytes + write_bytes},
            "census": census_all,
            "groups": {"size_hist": {str(k): v for k, v in sorted(size_hist.items())},
                       "wait_hist": {str(k): v for k, v in sorted(wait_hist.items())}},
            "gpu": torch.cuda.get_device_name(dev),
            "stats_exchange": {"READ": ex_tot[0], "WRITE": ex_tot[1], "decode_steps": ex_tot[2],
                               "note": "per-window async all_gather on a side stream, warm-up + timed windows"},
            "owners_all_ranks": {"n": len(versions_all), "versions": sorted(set(versions_all.values()))},
            "planner_host_share": plan_s / wall_s,
            "host_wall_ms_per_step": wall_s * 1e3 / a.steps,
            "clocks": clk.summary(),
            "config5_strong": c5,
            "config5_g8_rank_shape_on_1_gpu": c5_g8,
            "output_digest": {"sha256_by_rank": digests,
                              "what": "bf16 Y of every layer for the last timed window (all streams x C "
                                      "positions); fixed-order reductions: identical on reruns"},
        }
        if world == 1 and not a.no_cpu_baseline:
            from threadpoolctl import threadpool_limits

            sampler = OracleSample(1)
            cb = sampler()
            cb.pop("window_s", None)
            with threadpool_limits(limits=1):           # the 1-thread row beside it
                c1 = sampler()
            cb["one_thread"] = {"value": c1["value"], "unit": c1["unit"], "cores": 1,
                                "sample": "the same sample with BLAS limited to 1 thread (threadpoolctl)"}
            out["cpu_baseline"] = cb
            out["parity"] = sampled_parity(par_samples)
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
