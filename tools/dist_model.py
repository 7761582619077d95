"""Exchange volume and counts of the row-strip decomposed solve per inner (coarse-solve) step, and
the replicated coarse-level work, for configs[4]'s weak and strong families at N = 1..8 (DESIGN.md
§7).  Host arithmetic only: level sizes follow the hierarchy (n -> (n - 1) / 2 for Dirichlet),
decomposed levels 0..D (bench: D = 2), halos of 6 rows, one neighbour above and below.

Per inner step of the one-vector coarse FGMRES on level 1 (the decomposed path's exchange
schedule, helm.cu / dist.cuh): halos before the V-cycle's down legs of the decomposed levels
1..D and before E (fresh-ghost rule: one halo per decomposed level + E's), one all-gather of
level D + 1 after the level-D down leg, two rank sums (pass-1 dots, |w'|^2).  s-step form
(reading R28): the same halos per step, one rank sum of the block partials per s steps.
"""
import json


def levels(nx, ny, cut=512):
    out = [(nx, ny)]
    while True:
        nx2, ny2 = (nx - 1) // 2, (ny - 1) // 2
        if nx2 < 1 or ny2 < 1:
            break
        out.append((nx2, ny2))
        nx, ny = nx2, ny2
        if nx * ny <= cut:
            break
    return out


def model(kind, N, D=2, s=8, nvlink_gbs=900.0, op_us=8.0):
    if kind == "weak":   # N unit squares stacked in y, 2047 x 2048 per GPU (reading R27)
        nx, ny = 2047, 2048 * N - 1
    else:                # strong: 8191^2 split in N strips
        nx, ny = 8191, 8191
    lv = levels(nx, ny)
    halo_b = [6 * l[0] * 16 * (2 if N > 2 else 1) for l in lv]     # bytes received per rank per halo
    halos = list(range(1, D + 1)) + [1]                             # V-cycle levels 1..D + E on level 1
    halo_bytes = sum(halo_b[l] for l in halos) if N > 1 else 0
    gather_bytes = (lv[D + 1][0] * lv[D + 1][1] * 16 * (N - 1) // N) if N > 1 else 0
    ops_1v = (len(halos) + 1 + 2) if N > 1 else 0
    ops_ss = (len(halos) + 1 + 1.0 / s) if N > 1 else 0
    own1 = lv[1][0] * lv[1][1] / N                                  # level-1 unknowns per rank
    repl = sum(a * b for a, b in lv[D + 1:])                       # replicated unknowns (every rank)
    t_bytes = (halo_bytes + gather_bytes) / (nvlink_gbs * 1e3)      # us
    return {"kind": kind, "N": N, "grid": f"{nx}x{ny}", "level1_per_rank": int(own1),
            "replicated_unknowns": int(repl), "replicated_vs_owned_level1": round(repl / own1, 3),
            "halo_KB_per_step": round(halo_bytes / 1e3, 1), "allgather_KB_per_step": round(gather_bytes / 1e3, 1),
            "transfer_us_at_900GBs": round(t_bytes, 2),
            "collectives_per_step_one_vector": ops_1v, "collectives_per_step_sstep": round(ops_ss, 3),
            "latency_us_one_vector": round(ops_1v * op_us, 1), "latency_us_sstep": round(ops_ss * op_us, 1)}


if __name__ == "__main__":
    for kind in ("weak", "strong"):
        for N in (1, 2, 4, 8):
            print(json.dumps(model(kind, N)))
