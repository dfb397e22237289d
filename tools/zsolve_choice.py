"""Cut-axis line solves across P ranks: the paper's Schur partition (built) against an
all-to-all transpose that makes every z-line rank-local (SURVEY.md §8(e) "measure both").

Measured on one GPU:
  * Schur, as built: the device time of the two cut-axis phases (last Douglas sweep,
    divergence + first psi factor) on P emulated slabs (EMULATE transport: the same
    per-slab kernels, masters and exchanges, slabs run one after the other), divided
    by P = one rank's share; the single-GPU phases / P are the ideal.
  * transpose: the two on-device repacks every transposed field needs on each rank
    (pack the slab into P destination blocks of N/P rows, unpack the received blocks
    into full-length z-lines), timed as strided device copies of one rank's slab.
Counted from the implementation: the bytes each option puts on NVLink per rank and
step.  The NVLink time is that count over the per-direction NVSwitch bandwidth
(900 GB/s, an assumption: this run has one GPU), so it is an estimate, not a timing.

  python tools/zsolve_choice.py [cfg ...]      (default 3 4)
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1305_3976_b200 import ibgm, inputs  # noqa: E402

NVLINK_GBS = 900.0
CUT_PHASES = ("sweep_z", "div_psi_first")


def phase_ms(pr, steps, **kw):
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    ctx = ibgm.from_problem(pr, stream=st.cuda_stream, **kw)
    ctx.step(2)
    ctx.sync()
    ctx.set_profiling(True)
    ctx.step(steps)
    ctx.sync()
    ph = ctx.phase_times()
    ctx.close()
    return {k: ph[k][0] / ph[k][1] for k in CUT_PHASES}


def repack_ms(nz, n, P, reps=20):
    """pack [nz][n][n] -> [P][nz][n/P][n] and unpack [P][nz][n/P][n] -> [n/P][n][n]
    (full z for a block of rows): one field, one rank"""
    x = torch.randn(nz, n, n, dtype=torch.float64, device="cuda")
    recv = torch.empty(P, nz, n // P, n, dtype=torch.float64, device="cuda")
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    for _ in range(3):
        recv.copy_(x.view(nz, P, n // P, n).transpose(0, 1))
        recv.permute(2, 0, 1, 3).contiguous()
    torch.cuda.synchronize()
    e[0].record()
    for _ in range(reps):
        recv.copy_(x.view(nz, P, n // P, n).transpose(0, 1))
    e[1].record()
    for _ in range(reps):
        recv.permute(2, 0, 1, 3).contiguous()
    e[2].record()
    torch.cuda.synchronize()
    return e[0].elapsed_time(e[1]) / reps, e[1].elapsed_time(e[2]) / reps


def main():
    cfgs = [int(a) for a in sys.argv[1:]] or [3, 4]
    rows = []
    for cfg in cfgs:
        pr = inputs.config(cfg)
        if pr.dim != 3:
            continue
        n = pr.n
        steps = 20 if n <= 128 else 5
        single = phase_ms(pr, steps)
        for P in (2, 4, 8):
            nz = n // P
            plane = n * n
            emu = phase_ms(pr, steps, nranks=P, transport=ibgm.IB_TRANSPORT_EMULATE)
            # Schur bytes per rank and step (slab.cu: Q parts per slab, ns slots out,
            # nb = Q + 2 values per line and component back), off-rank share (P-1)/P
            Q = 1
            while Q < nz and (plane * Q < 65536 or nz % Q != 0):
                Q += 1
                while Q < nz and nz % Q != 0:
                    Q += 1
                if plane * Q >= 65536:
                    break
            if nz // Q < 2:
                Q = nz // 2
            Q = max(1, min(Q, 128 // P))
            while nz % Q:
                Q -= 1
            nb = Q + 2
            schur_doubles = Q * 6 * plane + 3 * nb * plane + Q * 4 * plane + 1 * nb * plane
            schur_mb = schur_doubles * 8 * (P - 1) / P / 1e6
            # transpose: 6 fields forward for the viscous z-sweep (increments, u^n), 3 back
            # (u^{n+1}); psi: 1 forward (RHS), 1 back
            nfield = 11
            field_mb = nz * plane * 8 / 1e6
            tr_mb = nfield * field_mb * (P - 1) / P
            pk, un = repack_ms(nz, n, P)
            row = {
                "cfg": cfg, "n": n, "P": P, "Q": Q,
                "schur_ms_per_rank": round(sum(emu.values()) / P, 4),
                "ideal_ms_per_rank": round(sum(single.values()) / P, 4),
                "schur_nvlink_mb": round(schur_mb, 2),
                "schur_nvlink_ms_est": round(schur_mb / 1e3 / NVLINK_GBS * 1e3, 4),
                "transpose_repack_ms": round(nfield * (pk + un), 4),
                "transpose_nvlink_mb": round(tr_mb, 1),
                "transpose_nvlink_ms_est": round(tr_mb / 1e3 / NVLINK_GBS * 1e3, 4),
            }
            # per rank: Schur = its measured passes + its exchanges; transpose = the local
            # single-GPU passes on 1/P of the lines + the repacks + its transfers
            row["schur_total_ms_est"] = round(row["schur_ms_per_rank"] + row["schur_nvlink_ms_est"], 4)
            row["transpose_total_ms_est"] = round(
                row["ideal_ms_per_rank"] + row["transpose_repack_ms"] + row["transpose_nvlink_ms_est"], 4)
            rows.append(row)
            print(json.dumps(row), flush=True)
    return rows


if __name__ == "__main__":
    main()
