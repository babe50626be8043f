"""Mutation check of the oracle's pins: each mutation below plants one plausible mistake in
`oracle/` (a dropped term, a wrong sign or index, a transposed operand, an off-by-one, a wrong
rounding or ordering rule) and the CPU suite (`pytest tests -m "not gpu"`) must FAIL for it.
A mutation that survives marks a part of the oracle no pin covers.

    python tools/oracle_mutations.py [--only NAME] > profiles/r2/oracle_mutations.txt

The oracle file is restored after every run (also on interrupt).  CPU only; ~35 s per mutation.
"""
from __future__ import annotations

import argparse
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (name, file, exact original text, mutated text)
MUTATIONS = [
    ("widen_bf16_low_bit", "oracle/numerics.py",
     "u = np.asarray(a, dtype=np.uint16).astype(np.uint32) << np.uint32(16)",
     "u = (np.asarray(a, dtype=np.uint16) ^ np.uint16(1)).astype(np.uint32) << np.uint32(16)"),
    ("round_bf16_ties_away", "oracle/numerics.py",
     "r = np.rint(np.ldexp(x[fin], -q))",
     "r = np.sign(x[fin]) * np.floor(np.abs(np.ldexp(x[fin], -q)) + 0.5)"),
    ("to_storage_skips_fp32_step", "oracle/numerics.py",
     "return round_bf16(np.asarray(x, dtype=np.float64).astype(np.float32).astype(np.float64))",
     "return round_bf16(np.asarray(x, dtype=np.float64))"),
    ("read_drops_delta", "oracle/numerics.py",
     "return (w_down + delta) @ z", "return w_down @ z"),
    ("read_rule1_drops_identity", "oracle/numerics.py",
     "return z + delta @ z", "return delta @ z"),
    ("write_eta_sign", "oracle/numerics.py",
     "cand = delta + eta * (V.T @ Z)", "cand = delta - eta * (V.T @ Z)"),
    ("write_last_token_only", "oracle/numerics.py",
     "cand = delta + eta * (V.T @ Z)", "cand = delta + eta * (V[-1:].T @ Z[-1:])"),
    ("write_rule1_drops_first_token", "oracle/numerics.py",
     "m = Z.sum(axis=0) / Z.shape[0]\n        cand", "m = Z[1:].sum(axis=0) / Z.shape[0]\n        cand"),
    ("lowrank_read_drops_delta", "oracle/lowrank.py",
     "return w_down @ z + B.T @ (A @ z)", "return w_down @ z"),
    ("lowrank_write_transposed", "oracle/lowrank.py",
     "A_new = A + eta * np.outer(A @ m, m)", "A_new = A + eta * np.outer(A @ m, m)[:, ::-1]"),
    ("lowrank_write_updates_b", "oracle/lowrank.py",
     "return nm.to_storage(A_new, dtype), np.array(B, copy=True)",
     "return nm.to_storage(A_new, dtype), nm.to_storage(B * (1 + eta), dtype)"),
    ("state_write_effect_one_early", "oracle/state.py",
     "return WRITE if self.tail_len(r) == self.C - 1 else READ",
     "return WRITE if self.tail_len(r) == self.C - 2 else READ"),
    ("state_rollback_keeps_tail", "oracle/state.py",
     "o.S = _copy(o.ckpt[1])\n        o.tail_z, o.tail_v, o.tail_p = [], [], []",
     "o.S = _copy(o.ckpt[1])"),
    ("state_rollback_keeps_version", "oracle/state.py",
     "o.v = o.ckpt[0]\n", "pass\n"),
    ("state_commit_bumps_two", "oracle/state.py",
     "o.v += 1", "o.v += 2"),
    ("state_fork_keeps_no_state", "oracle/state.py",
     "self.owners[dst] = Owner(v=o.v, S=_copy(o.S))",
     "self.owners[dst] = Owner(v=o.v, S=[np.zeros_like(x) if not isinstance(x, tuple) else tuple(np.zeros_like(y) for y in x) for x in o.S])"),
    ("prefill_tail_drops_first", "oracle/state.py",
     "for zs, vs, p in zip(zs_list, vs_list, ps):",
     "for zs, vs, p in list(zip(zs_list, vs_list, ps))[1:]:"),
    ("run_batched_ignores_failure", "oracle/run.py",
     "tab.write_group(list(g.owners), fail=fail)", "tab.write_group(list(g.owners), fail=False)"),
    ("run_retry_skipped", "oracle/run.py",
     "                    for s in ss:                            # fallback: serial singletons in μ order\n"
     "                        _retry(tab, rec, tr.owner(s), s, pos[s], vb[s])",
     "                    pass"),
    ("run_final_failure_keeps_chunk", "oracle/run.py",
     "        tab.drop_chunk(r)\n", "        pass\n"),
    ("planner_tiebreak_owner_first", "oracle/planner.py",
     "b = sorted(self.buckets[key], key=lambda e: (e.ready_step, e.owner))",
     "b = sorted(self.buckets[key], key=lambda e: (e.owner, e.ready_step))"),
    ("planner_wait_off_by_one", "oracle/planner.py",
     "if b and clock - b[0].ready_step >= self.w:",
     "if b and clock - b[0].ready_step > self.w:"),
    ("planner_arrival_no_version_check", "oracle/planner.py",
     "if V(e.owner) is None or e.version != V(e.owner):", "if V(e.owner) is None:"),
    ("planner_no_injectivity", "oracle/planner.py",
     "elif e.owner in pend:", "elif False:"),
    ("planner_no_version_check", "oracle/planner.py",
     "(keep if V(e.owner) == e.version else rejected).append(e)",
     "keep.append(e)"),
]


def run_suite() -> tuple[int, str]:
    r = subprocess.run([sys.executable, "-m", "pytest", "tests", "-m", "not gpu", "-x", "-q", "-p", "no:cacheprovider"],
                       cwd=ROOT, capture_output=True, text=True, timeout=1200)
    tail = [ln for ln in r.stdout.splitlines() if ln.strip()][-1:] or [""]
    return r.returncode, tail[0]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default=None)
    a = ap.parse_args()
    survived = 0
    for name, rel, old, new in MUTATIONS:
        if a.only and name != a.only:
            continue
        path = os.path.join(ROOT, rel)
        src = open(path).read()
        if src.count(old) != 1:
            print(f"{name:32s} SKIP (anchor not found once in {rel})")
            continue
        t0 = time.time()
        try:
            open(path, "w").write(src.replace(old, new))
            rc, tail = run_suite()
        finally:
            open(path, "w").write(src)
        verdict = "caught" if rc != 0 else "SURVIVED"
        survived += rc == 0
        print(f"{name:32s} {verdict:8s} ({time.time() - t0:.0f} s; {tail})", flush=True)
    print(f"survivors: {survived}")
    return 1 if survived else 0


if __name__ == "__main__":
    sys.exit(main())
