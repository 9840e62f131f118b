"""CPU model of the dual-GEMM persistent schedule (data-parallel tiles + a
stream-K tail, csrc/dual_gemm.cuh `Sched` / `sk_owner` and the host-side
split in csrc/cuasm_ffn.cu `launch_gemm`).  Checks, over many shapes, the
properties the kernel's correctness rests on:
  * every (tile, k-block) is computed exactly once;
  * each tile has exactly one owner of its last k-block (whole or finisher);
  * a finisher's contributor set (non-empty ranges from the owner of the
    tile's first k-block up to the cluster below it) is exactly the set of
    clusters that publish a partial of that tile, and each contributing
    cluster publishes at most once (one workspace slot per cluster), as the
    first segment it walks;
  * contributors never wait and finishers wait only for LOWER cluster ids
    (CTAs dispatched earlier), so the wait graph is acyclic and needs no
    co-residency of the grid.
"""
import itertools

import pytest


def plan(T, KB, max_clusters, schedule=0):
    clusters = min(T, max_clusters)
    sk_tiles = 0
    waves, rem = divmod(T, max_clusters)
    if schedule != 1 and KB > 1:
        if schedule == 2:
            sk_tiles = T
        elif rem != 0 and schedule == 3:
            sk_tiles = T if waves == 0 else rem
        elif rem != 0:
            sk_tiles = T if waves == 0 else rem + max_clusters
        if sk_tiles > 0:
            clusters = min(max_clusters, sk_tiles * KB)
            if schedule == 0 and waves == 0:
                clusters = min(clusters, (3 if T <= 32 else 2) * sk_tiles)   # kFewTiles / kFewTilesSplit
    return clusters, T - sk_tiles, sk_tiles * KB


def sk_begin(I, C, c):
    return (I * c) // C


def sk_owner(I, C, i):
    c = (i * C) // max(I, 1)
    while c + 1 < C and sk_begin(I, C, c + 1) <= i:
        c += 1
    while c > 0 and sk_begin(I, C, c) > i:
        c -= 1
    return c


def segments(cluster, C, KB, T_dp, I):
    t = cluster
    while t < T_dp:
        yield (t, 0, KB)
        t += C
    beg, cur = sk_begin(I, C, cluster), sk_begin(I, C, cluster + 1)
    while cur > beg:   # the stream-K range is walked backwards
        tt = (cur - 1) // KB
        lo = max(tt * KB, beg)
        yield (T_dp + tt, lo - tt * KB, cur - tt * KB)
        cur = lo


SHAPES = list(itertools.product([1, 2, 5, 8, 16, 22, 86, 88, 96, 148, 176, 512, 688, 700, 3584],
                                [1, 2, 3, 16, 64, 128], [74, 148], [0, 1, 2, 3]))


@pytest.mark.parametrize("T,KB,maxc,sched", SHAPES)
def test_schedule_properties(T, KB, maxc, sched):
    C, T_dp, I = plan(T, KB, maxc, sched)
    assert 1 <= C <= maxc
    covered = {}
    publishes = {}
    finishers = {}
    for c in range(C):
        segs = list(segments(c, C, KB, T_dp, I))
        contrib_segs = [s for s in segs if s[2] < KB]
        assert len(contrib_segs) <= 1, "a cluster publishes at most one partial"
        if contrib_segs:
            # the contributing segment is the first stream-K segment the cluster walks
            first_sk = next(s for s in segs if s[0] >= T_dp)
            assert contrib_segs[0] == first_sk
            publishes[contrib_segs[0][0]] = publishes.get(contrib_segs[0][0], set()) | {c}
        for (t, kb0, kb1) in segs:
            assert 0 <= kb0 < kb1 <= KB
            for kb in range(kb0, kb1):
                assert (t, kb) not in covered, "k-block computed twice"
                covered[(t, kb)] = c
            if kb1 == KB and kb0 > 0:
                assert t >= T_dp
                tile_start = (t - T_dp) * KB
                c_first = sk_owner(I, C, tile_start)
                waits = {cc for cc in range(c_first, c) if sk_begin(I, C, cc) != sk_begin(I, C, cc + 1)}
                finishers[t] = (c, waits)
                # the finisher's segment is the last one it walks
                assert (t, kb0, kb1) == segs[-1]
    assert len(covered) == T * KB
    for t in range(T):
        owner_last = covered[(t, KB - 1)]
        if t in finishers:
            c, waits = finishers[t]
            assert owner_last == c
            assert waits == publishes.get(t, set()), (t, waits, publishes.get(t))
            assert all(w < c for w in waits)
        else:
            assert t not in publishes, "partials published for a tile nobody finishes"
            assert all(covered[(t, kb)] == owner_last for kb in range(KB))


def test_7b_prefill_balance():
    # 2-SM: 8 m-blocks x 86 n-blocks, 64 k-blocks, 74 CTA pairs
    C, T_dp, I = plan(688, 64, 74)
    work = [sum(kb1 - kb0 for _, kb0, kb1 in segments(c, C, 64, T_dp, I)) for c in range(C)]
    assert max(work) - min(work) <= 1
    assert max(work) == -(-688 * 64 // 74)   # ceil: 9.30 tile-equivalents per pair, not 10


# ---- shape-keyed configuration model (csrc/cuasm_ffn.cu plan_config) ---------

def bn_frac(bn):
    return (1.0 if bn >= 128 else 0.925 if bn >= 120 else 0.867 if bn >= 112 else 0.80 if bn >= 96 else
            0.70 if bn >= 80 else 0.62)


TALL_FRAC = 1.07   # tall 80-wide k-block relative to a 128-wide 256-row one (csrc kTallFrac)


def plan_config(M, K, N, esize=2, sm_count=148, out_cols=128):
    t_kb, fixup, hbm, pen_1sm = 0.37e-6, 10e-6, 6.5e12, 1.16
    BK = 128 // esize
    KB = -(-K // BK)
    hbm_floor = ((2.0 if out_cols == 128 else 1.0) * N * K + M * K + M * N) * esize / hbm
    t1 = -(-M // 128) * -(-N // 128)
    t64 = -(-M // 128) * -(-N // 64)
    tall_ok = out_cols == 128 and esize == 2 and 256 < M <= 384   # tall tiles (csrc kTallBN = 80)
    if out_cols == 128 and esize == 2 and KB >= 48 and M <= 32 and 2 * t64 <= sm_count:
        return ("1sm", False, 256, 3 if 3 * t64 <= sm_count else 2, 64)   # decode shards, 64-wide tiles
    if out_cols == 128 and KB >= 48 and M <= 32:   # decode shards: cluster split-K
        S = (6 if M <= 16 and 6 * t1 <= sm_count and t1 <= 16 else
             4 if 4 * t1 <= sm_count and t1 <= 37 else
             3 if M <= 16 and 3 * t1 <= sm_count and t1 <= 49 else
             2 if 2 * t1 <= sm_count and t1 <= 64 else 0)
        if S:
            return ("1sm", False, 256, S, 128)
    few = KB >= 48 and ((M <= 256 and t1 <= 32) or (M <= 512 and t1 <= 64))
    small_m = out_cols == 128 and esize == 2 and few and M > 32   # small-M TP shards (profiles/r02/tune/grid.json)
    if small_m:
        if 2 * t64 <= sm_count:   # push-form splits (2 or 4 fit its slots)
            return ("1sm", False, 256, 4 if 4 * t64 <= sm_count else 3 if (M <= 64 and 3 * t64 <= sm_count) else 2, 64)
        if 2 * (-(-M // 256) * -(-N // 64)) <= sm_count // 2:
            return ("2sm", True, 256, 0, 64)
        if -(-M // 256) * -(-N // 80) <= sm_count // 2:
            return ("2sm", False, 256, 0, 80)
    if out_cols == 128 and few and not small_m:
        return ("1sm", True, 256, 0, 128)   # few-tile decode shapes (csrc kFewTiles / kFewTilesSplit)
    if KB <= 32 and out_cols != 128 and -(-M // 256) * -(-N // 128) <= sm_count // 2:   # GEMM mode, short k, one 2-SM wave
        return ("2sm", False, 128, 0, 128)
    best, best_t = ("2sm", False, 256, 0, 128), 1e30
    if out_cols == 128:   # SwiGLU tile widths (narrower than 128: 2-SM bf16 only)
        cands = [(256, bn) for bn in (128, 120, 112, 96, 80, 64) if bn == 128 or (esize == 2 and M > (32 if small_m else 128))]
    else:
        cands = [(256, 128), (128, 128)]
    for tn, bn in cands:
        oc = bn if out_cols == 128 else tn
        wrows = 2 * bn if out_cols == 128 else tn
        frac = bn_frac(bn) if out_cols == 128 else (1.0 if tn == 256 else 0.72)
        nblk = -(-N // oc)
        for cg in (2, 1):
            if bn != 128 and cg == 1:
                continue
            units = sm_count // cg
            mblk = -(-M // (128 * cg))
            tiles = mblk * nblk
            rounds = -(-tiles // units)
            pen = (pen_1sm if cg == 1 else 1.0) * frac
            t_dp = max(hbm_floor, rounds * KB * t_kb * pen)
            rem = tiles % units
            sk_tiles = tiles if tiles < units else (rem + units if rem else 0)
            gm = min(mblk, max(1, min(16, (32 << 20) // (128 * cg * K * esize))))
            region = (-(-sk_tiles // gm) + 1) * wrows * K * esize + min(M, gm * 128 * cg) * K * esize
            l2_pen = 1.32 if region > 120e6 else 1.0
            sk_units = min(units, 2 * tiles) if tiles < units else units
            t_sk = max(hbm_floor, tiles * KB * t_kb * pen * l2_pen / sk_units + fixup)
            name = "2sm" if cg == 2 else "1sm"
            if t_dp < best_t * 0.999:
                best_t, best = t_dp, (name, False, tn, 0, bn)
            if K // BK > 1 and t_sk < best_t * 0.98:
                best_t, best = t_sk, (name, True, tn, 0, bn)
    if tall_ok:
        t_tall = max(hbm_floor, -(-(-(-N // 80)) // (sm_count // 2)) * KB * t_kb * TALL_FRAC)
        if t_tall < best_t * 0.98:
            best = ("tall", False, 256, 0, 80)
    return best


# Best measured configuration per M at K=4096, N=11008 (profiles/r01/tune.json,
# B200; "auto" there was the hybrid 2-SM stream-K tail).  Where two
# configurations were within 2% the model may pick either.
MEASURED_BEST = {
    16: {("1sm", False)},
    128: {("1sm", False)},
    192: {("2sm", True)},
    256: {("2sm", True)},
    384: {("1sm", False)},
    512: {("2sm", True)},
    768: {("2sm", True), ("2sm", False)},
    1024: {("2sm", False)},
    1536: {("2sm", False)},
    2048: {("2sm", True)},
    4096: {("2sm", True), ("2sm", False)},
}


@pytest.mark.parametrize("M", sorted(MEASURED_BEST))
def test_plan_matches_measured_best(M):
    # (a table of 128-wide configurations: shapes whose plan takes a narrower tile are
    # checked against profiles/r02/tune_bn.json below)
    pl = plan_config(M, 4096, 11008)
    assert pl[4] != 128 or pl[:2] in MEASURED_BEST[M]


def test_plan_70b_shard_uses_narrow_whole_tiles():
    # 8-way shard of the 70B FFN: 448 128-wide tiles = 6.05 waves of 74 CTA pairs (stream-K
    # 292.5 us) vs 512 112-wide tiles = 6.92 waves (whole tiles 282.4 us, profiles/r02/tune_bn.json)
    assert plan_config(4096, 8192, 3584) == ("2sm", False, 256, 0, 112)


def test_plan_w2_down_projection_avoids_l2_thrashing_stream_k():
    # hidden [2048, 11008] x W2 [4096, 11008]: whole tiles 128 us vs stream-K 158 us measured
    # (256-wide stream-K would thrash L2: 128 us whole tiles vs 158 us measured)
    assert plan_config(2048, 11008, 4096, out_cols=256)[:3] != ("2sm", True, 256)


# ---- the library's own implementation agrees with the model above -------------------
@pytest.fixture(scope="module")
def lib_plan():
    from paper_2501_08071_b200 import build as ffn_build
    ffn_build.build()
    import paper_2501_08071_b200 as ffn
    return ffn.plan_config


@pytest.mark.parametrize("M", sorted(MEASURED_BEST))
def test_library_plan_matches_measured_best(lib_plan, M):
    pl = lib_plan(M, 4096, 11008)
    assert pl[4] != 128 or pl[:2] in MEASURED_BEST[M]


@pytest.mark.parametrize("M,K,N,op", [(m, k, n, op) for m in (1, 16, 200, 512, 1000, 2048, 4096, 16384)
                                      for k, n in ((4096, 11008), (8192, 3584), (11008, 4096), (2048, 512), (4096, 1376))
                                      for op in ("ffn", "gemm")])
def test_library_plan_equals_python_mirror(lib_plan, M, K, N, op):
    assert lib_plan(M, K, N, op) == plan_config(M, K, N, out_cols=128 if op == "ffn" else 256)


def test_plan_paper_mmleakyrelu_is_whole_tiles(lib_plan):
    # 512 x 2048 x 512: 4 tiles of 2-SM; stream-K would split each tile many ways
    assert lib_plan(512, 2048, 512, "gemm")[1] is False


# measured best of {1-SM, 2-SM} x {whole tiles, stream-K} x {256, 128 wide} for the
# GEMM + activation mode (profiles/r01/tune_gemm*.log); near-ties (<= 3%) accept either
GEMM_MEASURED = {
    (512, 4096, 4096): {("2sm", False, 128)},
    (2048, 4096, 4096): {("2sm", False, 256)},
    (4096, 4096, 4096): {("2sm", False, 256), ("2sm", True, 256)},
    (8192, 4096, 4096): {("2sm", False, 256)},
    (2048, 11008, 4096): {("2sm", False, 256)},
    (4096, 11008, 4096): {("2sm", False, 256)},
    (512, 2048, 512): {("2sm", False, 128), ("2sm", False, 256)},
    (4096, 2048, 512): {("2sm", False, 128), ("2sm", False, 256)},   # (r02: 20.5 vs 1-SM 22.6 us)
    (512, 11008, 4096): {("2sm", True, 256), ("1sm", True, 256)},
}


@pytest.mark.parametrize("shape", sorted(GEMM_MEASURED))
def test_library_gemm_plan_matches_measured_best(lib_plan, shape):
    M, K, N = shape
    assert lib_plan(M, K, N, "gemm")[:3] in GEMM_MEASURED[shape]


def test_library_plan_w2_and_70b(lib_plan):
    assert lib_plan(2048, 11008, 4096, "gemm")[:3] != ("2sm", True, 256)
    assert lib_plan(4096, 8192, 3584) == ("2sm", False, 256, 0, 112)


# best measured SwiGLU tile width (profiles/r02/tune_bn.json, tune_bn120.json; near-ties <= 1.5%
# accept either)
BN_MEASURED = {
    (2048, 4096, 1376): {80},
    (2048, 4096, 2752): {112, 80},
    (2048, 4096, 5504): {120},
    (2048, 4096, 11008): {120},
    (1024, 4096, 1376): {80, 96},
    (1024, 4096, 2752): {80},
    (512, 4096, 11008): {112, 80},
    (1024, 4096, 11008): {120},
    (4096, 4096, 11008): {120},
    (16384, 4096, 11008): {120, 112},
    (256, 4096, 11008): {80},
    (4096, 8192, 3584): {112},
    (4096, 8192, 7168): {112, 120, 128},
    (4096, 8192, 14336): {112, 120, 128},
    (4096, 8192, 28672): {120, 112},
    (768, 4096, 11008): {120},
    (16384, 4096, 1376): {128},
}


@pytest.mark.parametrize("shape", sorted(BN_MEASURED))
def test_plan_tile_width_matches_measured_best(lib_plan, shape):
    assert plan_config(*shape)[4] in BN_MEASURED[shape]
    assert lib_plan(*shape)[4] in BN_MEASURED[shape]


# measured (profiles/r01/csplit/ncu_ab_*.txt, profiles/r02/tune_decode_bn.log): the cluster
# split-K wins on few-tile shards with M <= 32; with 64-output tiles (up to 74 of them) a split of
# 3 (2) beats the 128-output tile's; 65 128-wide tiles: no gain.  On 128-output tiles it loses at
# M >= 64 (pull-form reduction), but on 64-output tiles the autotuner found it best up to M = 128
# (profiles/r02/tune/grid.json: 64 x 4096 x 1376 18.7 us vs 21.9 for the 1-SM stream-K tile)
@pytest.mark.parametrize("M,K,N,cs,bn", [(16, 4096, 1376, 3, 64), (16, 4096, 2752, 3, 64), (16, 8192, 3584, 2, 64),
                                         (32, 4096, 1376, 3, 64), (1, 4096, 1376, 3, 64), (16, 4096, 5504, 3, 128),
                                         (32, 4096, 5504, 2, 128), (16, 4096, 6880, 2, 128),
                                         (16, 8192, 7168, 2, 128), (16, 4096, 8256, 0, 128),
                                         (64, 4096, 1376, 4, 64), (48, 4096, 2752, 3, 64), (128, 4096, 1376, 4, 64),
                                         (256, 4096, 1376, 2, 64), (384, 4096, 1376, 2, 64), (512, 4096, 1376, 0, 80),
                                         (96, 4096, 2752, 2, 64), (128, 8192, 3584, 2, 64),
                                         (16, 4096, 11008, 0, 128)])
def test_plan_cluster_split_for_decode_shards(lib_plan, M, K, N, cs, bn):
    assert plan_config(M, K, N)[3:] == (cs, bn)
    assert lib_plan(M, K, N)[3:] == (cs, bn)


# every cluster split the planner picks at M <= 128 must take the push form (dual_gemm.cuh split_k_push_fits:
# bf16, <= 32 rows, ceil(NU / S) * S * rc * 128 bytes of slots within the 32 KB staging area, NU =
# 2 BN / 16 units, rc = 16, 32, 64 or 128 slot rows, 64 KB of staging on the 1-SM 64-output tile); the pull
# form is only reachable by forcing CUASM_OPT_CSPLIT
@pytest.mark.parametrize("K", [4096, 8192])
def test_planner_cluster_splits_take_the_push_form(K):
    for M in list(range(1, 129)) + [160, 192, 256, 300, 384, 448, 512]:
        for n8 in range(1, 160):
            N = 64 * n8
            pl = plan_config(M, K, N)
            S, bn = pl[3], pl[4]
            if S:
                rc = 16 if M <= 16 else 32 if M <= 32 else 64 if M <= 64 else 128
                nu = 2 * bn // 16 // 2
                stg = 65536 if bn == 64 else 32768   # (the 1-SM 64-output tile's staging area is 64 KB)
                assert -(-nu // S) * S * rc * 128 <= stg, (M, N, S, bn)
                assert -(-N // bn) * S <= 148


# the small-M shard rules (32 < M <= 512, few tiles) against the autotuner's grid: the plan's measured
# time is within 10% of the best candidate's at every grid shape the rules cover, and never slower
# than the 1-SM stream-K tile they replaced (profiles/r02/tune/grid.json, L2-flushed, one B200)
def test_small_m_shard_rules_match_the_tuned_grid():
    import json
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    grid = json.load(open(os.path.join(root, "profiles", "r02", "tune", "grid.json")))
    checked = 0
    for r in grid["rows"]:
        M, K, N = r["M"], r["K"], r["N"]
        t1 = -(-M // 128) * -(-N // 128)
        if not (32 < M <= 512 and ((M <= 256 and t1 <= 32) or t1 <= 64)):   # the rules' few-tile region
            continue
        pl = list(plan_config(M, K, N))
        t = r["all"].get(str(pl))
        assert t is not None, (M, K, N, pl)
        assert t <= 1.10 * r["best_us"], (M, K, N, pl, t, r["best"], r["best_us"])
        if r["model"] == ["1sm", True, 256, 0, 128]:   # shapes the replaced rule used to take
            assert t <= r["model_us"] * 1.02, (M, K, N, pl, t, r["model_us"])
        checked += 1
    assert checked >= 25


# tall tiles (257..384 rows, bf16 SwiGLU; csrc kTallBN = 80): the flags word's bit 2, decoded by the
# binding as the variant name "tall"; the Python mirror agrees across the region's edges
@pytest.mark.parametrize("M", [256, 257, 288, 320, 384, 385])
def test_library_plan_tall_region(lib_plan, M):
    pl = lib_plan(M, 4096, 11008)
    assert pl == plan_config(M, 4096, 11008)
    assert (pl[0] == "tall") == (256 < M <= 384)
    if pl[0] == "tall":
        assert pl[1:] == (False, 256, 0, 80)
    import torch
    assert lib_plan(M, 4096, 11008, "ffn", torch.float32)[0] != "tall"   # fp32: no tall tiles
