"""Generate the explicit tile_kernel instantiations and their dispatch table.

Writes paper_2505_23618_b200/csrc/gen/inst_<k>.cu (one translation unit per
shard, compiled in parallel) and gen/registry.inc (the lookup table the C-ABI
searches).  Every instantiation is a (dtype, H, W, row-op, column-op,
direction, in/out addressing) tuple; the ops are the per-axis stage pairs of
butterfly.cuh.  Anything not listed here is served by the dense-composite
fallback in abi.cu (also listed, per shape).
"""
from __future__ import annotations

import os
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1] / "paper_2505_23618_b200" / "csrc" / "gen"
NSHARDS_HOT = 12   # gen/inst_hNN.cu: the configs' 2-D kernels, compiled with -lineinfo
NSHARDS_COLD = 12  # gen/inst_cNN.cu: 1-D primitives, dense composites, copy (no line info)
# Measured-slower tuning variants (DCTADJ_VARIANT=k) are built only with
# DCTADJ_TUNING=1; the shipped library holds the defaults alone.
TUNING = os.environ.get("DCTADJ_TUNING", "0") not in ("", "0")

NONE, DCT2, IDCT2, DST3, IDST3, BAND, SUB, DENSE, GIVENS_LIFT, GIVENS = range(10)
# GIVENS: the band's Givens schedule as scaled rotations (ST_GIVENS2, 2 FMAs per
# rotation); the lifting form (ST_GIVENS, 3 FMAs) is no longer instantiated


def code(s1, s2=NONE, k=0):
    return s1 | (s2 << 4) | (k << 8)


ID = code(NONE)

DTYPES = {"float": 0, "double": 1}


def tile_config(dtype: str, h: int, w: int, two_d: bool, col_first: bool = False,
                rc: int = 0):
    """(P blocks per super-tile, NG warps per CTA, S ring stages, pair_rows).

    Measured on B200 (back-to-back launches, profiles/r01_tuning.md): for 32x32
    fp32 both directions run best with 8 KB super-tiles (P=2) and 4 warps x 4
    stages per CTA; packed row pairs help everywhere except the inverse
    sub-block kernel, and the inverse band (Givens) kernel prefers 16 KB super-
    tiles with 2 warps x 3 stages."""
    es = 4 if dtype == "float" else 8
    p = 1
    pr = False
    if two_d:
        # rows: P*H >= 32; packed column pairs (fp32): P*W >= 64
        p = max(1, 32 // h, (64 // w) if dtype == "float" else 32 // w)
    if two_d and (rc & 15) == DENSE:
        # the dense comparison path is FMA-bound: many warps, scalar lanes; the
        # two dense matrices sit in shared memory beside the rings (<= 200 KB)
        p = max(1, 32 // h, 32 // w)
        stage = -(-(p * h * w * es) // 1024) * 1024
        dense = (h * h + w * w) * es
        for s in (3, 2):
            ng = min(8, (200 * 1024 - dense) // (s * stage))
            if ng >= 1:
                return p, ng, s, False
        raise ValueError(f"dense {h}x{w} {dtype} does not fit shared memory")
    small32 = two_d and dtype == "float" and h * w <= 1024
    band_inv = col_first and (rc >> 8) in (4, 6) and (rc & 15) != SUB and ((rc >> 4) & 15) in (BAND, GIVENS)
    if small32:
        if band_inv:
            p, ng, s, pr = max(p, 4 * 1024 // (h * w)), 2, 3, True
        else:
            p, ng, s, pr = max(p, 2 * 1024 // (h * w)), 4, 4, not col_first
        if (p * h) % 64 or (rc & 15) == DENSE:
            pr = False  # dense rows read shared-memory coefficients: keep scalar FFMA
        return p, ng, s, pr
    tile = p * h * w * es
    stage = -(-tile // 1024) * 1024
    if two_d and dtype == "float" and (h, w) == (64, 64):
        givens = (rc & 15) == GIVENS or ((rc >> 4) & 15) == GIVENS
        if givens:
            # band-6 pre (Givens): the shared-ring kernel -- 8 compute warps with
            # packed 64-point passes (168 registers: 3 warps share an SMSP) + a TMA
            # producer, 13 x 16 KB stages shared by the warps (ring_kernel, CH bit
            # 3).  Measured (profiles/r02_tuning.md) fwd / inv 1.62 / 1.65 ms vs
            # 1.82-1.87 / 1.75 for the two-warp scalar tile kernel; 7 warps at 188
            # registers 1.77 / 1.70; one butterfly copy for both passes 2.31 / 1.96
            return 1, 8, 13, ("RING", 1, 8)
        if col_first:
            # 64-point vectors: two warps per tile, scalar lanes, 12 warps/SM
            # (the packed 64-column pass needs ~200 registers; measured faster)
            return p, 6, 2, ("NW", 2, 0)
    if two_d and dtype == "double" and (h, w) == (32, 32):
        # fp64 32x32 (config 1): one-warp CTAs, one block per stage, two stages, 12
        # CTAs/SM (launch bounds) -> 12 warps/SM, no spills; small CTAs let the next
        # launch's CTAs become resident as these retire.  Measured 13.9 us per
        # 4,096-block forward vs 14.2 (two-warp groups on 2-block super-tiles, 6
        # CTAs/SM) and 16.9 (4 x 1 warp, 3 stages, 8 warps/SM); profiles/r01_tuning.md
        return 1, 1, 2, ("NW", 1, 0xC0)
    if stage <= 2048:
        ng, s = 8, 4
    elif stage <= 4096:
        ng, s = 8, 3
    elif stage <= 8192:
        ng, s = 4, 3
    elif stage <= 16384:
        ng, s = (4, 3) if two_d and dtype == "float" and (rc & 15) != GIVENS \
            and ((rc >> 4) & 15) != GIVENS else (6, 2)
    else:
        ng, s = 3, 2
    return p, ng, s, pr


def one_d_ops(n: int):
    ops = [code(DCT2), code(IDCT2), code(DST3), code(IDST3), code(DENSE)]
    ops += [code(BAND, k=4), code(BAND, DST3, 4), code(IDST3, BAND, 4),
            code(BAND, IDCT2, 4), code(DCT2, BAND, 4)]
    if n >= 8:
        ops += [code(BAND, k=6), code(SUB, k=8),
                code(BAND, DST3, 6), code(IDST3, BAND, 6),
                code(BAND, IDCT2, 6), code(DCT2, BAND, 6),
                code(DCT2, SUB, 8), code(SUB, IDCT2, 8)]
    # band as Givens lifting layers (schedule supplied), fused with the base
    for k in (4, 6):
        if k <= n:
            ops += [code(GIVENS, DST3, k), code(IDST3, GIVENS, k),
                    code(GIVENS, IDCT2, k), code(DCT2, GIVENS, k)]
    return ops


def two_d_pairs():
    """(row op, col op, col_first) for the fused 2-D kernels."""
    fwd = []
    inv = []
    fwd.append((code(DCT2, SUB, 8), code(DCT2, SUB, 8)))
    inv.append((code(SUB, IDCT2, 8), code(SUB, IDCT2, 8)))
    # band pre-adjustments run as Givens lifting layers in the fused 2-D kernels
    # (a band given only as a matrix falls back to the dense composite)
    for kh in (DST3, IDCT2):          # DST-7 (DST-3 base) / DCT-8 (DCT-3 base, R*A*R band)
        for kv in (DST3, IDCT2):
            fwd.append((code(GIVENS, kh, 6), code(GIVENS, kv, 6)))
            ih = IDST3 if kh == DST3 else DCT2
            iv = IDST3 if kv == DST3 else DCT2
            inv.append((code(ih, GIVENS, 6), code(iv, GIVENS, 6)))
    for kb in (DST3, IDCT2):
        fwd.append((code(GIVENS, kb, 4), code(GIVENS, kb, 4)))
        ib = IDST3 if kb == DST3 else DCT2
        inv.append((code(ib, GIVENS, 4), code(ib, GIVENS, 4)))
    fwd.append((code(DCT2), code(DCT2)))
    inv.append((code(IDCT2), code(IDCT2)))
    fwd.append((code(DENSE), code(DENSE)))
    inv.append((code(DENSE), code(DENSE)))
    return [(r, c, False) for r, c in fwd] + [(r, c, True) for r, c in inv]


def pair_flags(dt, h, w, p, rc, cc):
    """Default packing: fp32 column pairs (FFMA2) when a column op exists and
    the super-tile has >= 64 columns (not for the dense comparison path)."""
    if dt != "float" or cc == ID or (cc & 15) == DENSE:
        return (False, False)
    return (False, (p * w) % 64 == 0)


# tuning variants for the 32x32 fp32 hot kernels (DCTADJ_VARIANT=k): (P, NG, S)
# tuning variants (DCTADJ_VARIANT=k, k >= 1), per (H, W) of fp32 uniform 2-D kernels:
# (P, NG, S, pair_rows, pair_cols, L2 hints); variant 0 is always the default build
EXPERIMENT = {
    ("double", 32, 32): [(1, 8, 2, False, False, 0, 1), (1, 2, 4, False, False, 0, 1),
                         (2, 2, 2, False, False, 0, 2), (2, 3, 2, False, False, 0, 2),
                         (2, 1, 4, False, False, 0, 2), (1, 12, 2, False, False, 0, 1),
                         (2, 1, 3, False, False, 0, 2), (2, 1, 2, False, False, 0x60, 2),
                         (2, 1, 3, False, False, 0x50, 2), (4, 1, 3, False, False, 0, 4),
                         (4, 1, 2, False, False, 0x30, 4), (2, 1, 4, False, False, 0x40, 2),
                         (1, 6, 2, False, False, 0, 1), (2, 1, 5, False, False, 0, 2),
                         (2, 1, 2, False, False, 0x60, 2), (1, 1, 3, False, False, 0x80, 1)],
    ("float", 32, 32): [(4, 2, 3, True, True, 0), (2, 4, 4, True, True, 0), (4, 2, 3, False, True, 0),
               (2, 4, 4, False, True, 0)],
    ("float", 64, 64): [(1, 6, 2, False, False, 0, 2), (1, 4, 3, False, False, 0, 2),
               (1, 5, 2, False, False, 0, 2), (1, 3, 4, False, False, 0, 2),
               (2, 3, 2, False, False, 0, 4), (2, 2, 3, False, False, 0, 4),
               # shared-ring kernel (CH bit 3): NC compute warps x S stages
               (1, 7, 13, True, True, 8, 1), (1, 11, 13, True, True, 8, 1),
               (1, 11, 14, True, True, 8, 1)],
}
EXPERIMENT_OPS = None  # filled below: the band-6 and sub-8 2-D ops
# interleaved frame kernels (config 5): (P, NG, S); pair flags as the default
# mixed-shape gather kernels (config 3): (P multiplier, NG, S) relative to the default
GATHER_EXPERIMENT = [(1, 5, 2), (1, 7, 2), (2, 3, 2), (1, 4, 2), (1, 4, 3), (2, 2, 3)]
GATHER_BINV_EXPERIMENT = [(4, 2, 3), (2, 4, 3), (4, 3, 2), (4, 4, 2), (1, 8, 2), (2, 5, 2)]
FRAME_IL_EXPERIMENT = [(4, 2, 3), (2, 4, 6), (4, 3, 3), (4, 4, 2), (8, 2, 3)]


def instances():
    out = []
    for dt in DTYPES:
        for n in (4, 8, 16, 32, 64):
            for op in one_d_ops(n):
                p, ng, s, pr = tile_config(dt, 32, n, False)
                out.append((dt, 32, n, p, op, ID, False, 0, 0, ng, s, pr))
        shapes = [(16, 16), (16, 32), (32, 16), (32, 32), (64, 64)]
        if dt == "double":
            shapes = [(16, 16), (32, 32), (64, 64)]
        for h, w in shapes:
            for rc, cc, cf in two_d_pairs():
                p, ng, s, pr = tile_config(dt, h, w, True, cf, rc)
                out.append((dt, h, w, p, rc, cc, cf, 0, 0, ng, s, pr))
    # dense composite on every shape: the fallback that makes any (H, W) and any
    # per-axis op combination available as one fused 2-D kernel
    have = {(x[0], x[1], x[2], x[4], x[5], x[6]) for x in out}
    for dt in DTYPES:
        for h in (4, 8, 16, 32, 64):
            for w in (4, 8, 16, 32, 64):
                for cf in (False, True):
                    if (dt, h, w, code(DENSE), code(DENSE), cf) in have:
                        continue
                    p, ng, s, pr = tile_config(dt, h, w, True, cf, code(DENSE))
                    out.append((dt, h, w, p, code(DENSE), code(DENSE), cf, 0, 0, ng, s, pr))
    # frame tiling (config 5): 32x32 fp32, frames in / blocks out and back
    for rc, cc, cf in two_d_pairs():
        if rc == code(DCT2) or (rc >> 8) == 4:
            continue
        p, ng, s, pr = tile_config("float", 32, 32, True, cf, rc)
        in_mode, out_mode = (0, 1) if cf else (1, 0)
        out.append(("float", 32, 32, p, rc, cc, cf, in_mode, out_mode, ng, s, pr))
        # one-box-per-super-tile interleaved variant (frame width a multiple of P
        # blocks): 16 KB super-tiles (512-byte frame-row segments), 4 warps x 3
        # stages -- measured best on B200 (forward at the HBM roofline)
        in_mode, out_mode = (5, 4) if cf else (4, 5)
        out.append(("float", 32, 32, 4, rc, cc, cf, in_mode, out_mode, 4, 3, pr))
    # mixed-shape gather kernels (config 3): fp32, the four C3 shapes, pre + post
    for h, w in ((16, 16), (16, 32), (32, 16), (32, 32)):
        for rc, cc, cf in two_d_pairs():
            if rc in (code(DCT2), code(IDCT2)) or (rc >> 8) == 4:
                continue
            p, ng, s, pr = tile_config("float", h, w, True, cf, rc)
            # gather tiles (one box per block) want more groups in flight with fewer
            # stages each: 6 x 2 measured 13-25 % faster on config 3 than the
            # uniform kernels' choices (4 x 4; band inverse: 16 KB super-tiles, 2 x 3)
            if (ng, s) == (4, 4):
                ng, s = 6, 2
            elif (ng, s) == (2, 3):
                p, ng, s = 2 * 1024 // (h * w), 6, 2
            out.append(("float", h, w, min(p, 32), rc, cc, cf, 2, 2, ng, s, pr))
    # identity-op tile round trip (TMA in -> smem -> TMA out, no arithmetic):
    # the data-movement ceiling of the tile pipeline (dctadj_copy_tiles)
    for dt in DTYPES:
        for h, w in ((32, 32), (64, 64), (16, 16)):
            p, ng, s, pr = tile_config(dt, h, w, True)
            out.append((dt, h, w, p, ID, ID, False, 0, 0, ng, s, False))
    # attach packing flags + tuning variants (variant 0 = default)
    final = []
    for inst in out:
        dt, h, w, p, rc, cc, cf, im, om, ng, s_, pr = inst
        _, pc = pair_flags(dt, h, w, p, rc, cc)
        if isinstance(pr, tuple) and pr[0] == "NW":  # NW warps per tile, scalar lanes, CH bits
            final.append(inst[:11] + (False, False, 0, pr[2], pr[1]))
        elif isinstance(pr, tuple) and pr[0] == "RING":  # ring kernel: packed rows + columns
            final.append(inst[:11] + (True, True, 0, pr[2], pr[1]))
        else:
            final.append(inst[:11] + (pr and cc != ID, pc, 0, 0))
        if not TUNING:
            continue
        if (im, om) == (2, 2):
            binv = cf and (rc >> 8) in (4, 6) and (rc & 15) != SUB and ((rc >> 4) & 15) in (BAND, GIVENS)
            exps = GATHER_BINV_EXPERIMENT if binv else GATHER_EXPERIMENT
            for k, (pm, nng, ss) in enumerate(exps, start=1):
                # band-inverse entries give P in 32x32-block units (scaled to the shape)
                pp = min(max(1, pm * 1024 // (h * w)) if binv else p * pm, 32)
                if nng * ss * (-(-(pp * h * w * 4) // 1024) * 1024) > 200 * 1024:
                    continue  # does not fit shared memory: the default serves this variant
                _, ppc = pair_flags(dt, h, w, pp, rc, cc)
                ppr = pr and cc != ID and (pp * h) % 64 == 0
                final.append((dt, h, w, pp, rc, cc, cf, im, om, nng, ss, ppr, ppc, k, 0, 1))
        if (dt, h, w) == ("float", 32, 32) and (im, om) in ((4, 5), (5, 4)):
            for k, (pp, nng, ss) in enumerate(FRAME_IL_EXPERIMENT, start=1):
                _, ppc = pair_flags(dt, h, w, pp, rc, cc)
                final.append((dt, h, w, pp, rc, cc, cf, im, om, nng, ss, pr and cc != ID, ppc, k, 0, 1))
        if (dt, h, w) in EXPERIMENT and im == 0 and om == 0 and rc == cc \
                and rc in (code(DCT2, SUB, 8), code(SUB, IDCT2, 8), code(GIVENS, DST3, 6),
                           code(IDST3, GIVENS, 6)):
            for k, ex in enumerate(EXPERIMENT[(dt, h, w)], start=1):
                pp, nng, ss, pr, pc, ch = ex[:6]
                nw = ex[6] if len(ex) > 6 else 1
                final.append((dt, h, w, pp, rc, cc, cf, im, om, nng, ss, pr, pc, k, ch, nw))
    return final


def _targs(inst) -> str:
    dt, h, w, p, rc, cc, cf, im, om, ng, s, pr, pc, var, ch = inst[:15]
    nw = inst[15] if len(inst) > 15 else 1
    b = lambda v: "true" if v else "false"  # noqa: E731
    return (f"{dt}, {h}, {w}, {p}, {rc}, {cc}, {b(cf)}, {im}, {om}, {ng}, {s}, {b(pr)}, {b(pc)}, "
            f"{ch}, {nw}")


def _write_if_changed(path: Path, text: str) -> None:
    """Keep timestamps (and make's incremental build) when nothing changed."""
    if not path.exists() or path.read_text() != text:
        path.write_text(text)


def is_hot(inst) -> bool:
    """The BASELINE configs' 2-D kernels -- built with -lineinfo so ncu's source
    page maps onto them: every gather (C3) and frame (C5) kernel, and the linear
    fp32 32x32 / 64x64 and fp64 32x32 kernels of the sub-8 post and same-kind
    band-6 (Givens) pre pairs (C1, C2, C4)."""
    dt, h, w, p, rc, cc, cf, im, om = inst[:9]
    if cc == ID or rc == code(DENSE):
        return False  # 1-D primitives, copy tiles, dense composites
    if (im, om) != (0, 0):
        return True
    if (dt, h, w) not in (("float", 32, 32), ("float", 64, 64), ("double", 32, 32)):
        return False
    sub = {code(DCT2, SUB, 8), code(SUB, IDCT2, 8)}
    g6 = {code(GIVENS, DST3, 6), code(IDST3, GIVENS, 6), code(GIVENS, IDCT2, 6),
          code(DCT2, GIVENS, 6)}
    return rc == cc and (rc in sub or rc in g6)


def main():
    ROOT.mkdir(parents=True, exist_ok=True)
    insts = instances()
    hot = [[] for _ in range(NSHARDS_HOT)]
    cold = [[] for _ in range(NSHARDS_COLD)]
    seen = set()
    nh = nc = 0
    for inst in insts:
        if _targs(inst) in seen:  # a tuning variant equal to a default: one definition
            continue
        seen.add(_targs(inst))
        if is_hot(inst):
            hot[nh % NSHARDS_HOT].append(inst)
            nh += 1
        else:
            cold[nc % NSHARDS_COLD].append(inst)
            nc += 1
    reg = ["// Generated by tools/gen_instances.py -- do not edit.",
           f"// {len(insts)} tile_kernel instantiations ({nh} hot, {nc} cold)"
           f"{' + tuning variants' if TUNING else ''}."]
    wanted = set()
    for tag, shards in (("h", hot), ("c", cold)):
        for k, shard in enumerate(shards):
            lines = ["// Generated by tools/gen_instances.py -- do not edit.",
                     '#include "../launch.cuh"', "", "namespace dctadj {", ""]
            for inst in shard:
                lines.append(f"template int launch_tile<{_targs(inst)}>(const LaunchArgs&);")
            lines += ["", "}  // namespace dctadj", ""]
            name = f"inst_{tag}{k:02d}.cu"
            wanted.add(name)
            _write_if_changed(ROOT / name, "\n".join(lines))
    for stale in ROOT.glob("inst_*.cu"):
        if stale.name not in wanted:
            stale.unlink()
    decl = []
    rows = []
    declared = set()
    for inst in insts:
        dt, h, w, p, rc, cc, cf, im, om, ng, s, pr, pc, var, ch = inst[:15]
        targs = _targs(inst)
        if targs not in declared:
            declared.add(targs)
            decl.append(f"extern template int launch_tile<{targs}>(const LaunchArgs&);")
        rows.append(f"  {{{DTYPES[dt]}, {h}, {w}, {rc}, {cc}, {int(cf)}, {im}, {om}, {var}, "
                    f"&launch_tile<{targs}>}},")
    reg += decl + ["", "static const KernelEntry kRegistry[] = {"] + rows + ["};", ""]
    _write_if_changed(ROOT / "registry.inc", "\n".join(reg))
    print(f"{len(insts)} instantiations: {nh} hot + {nc} cold in "
          f"{NSHARDS_HOT} + {NSHARDS_COLD} shards")


if __name__ == "__main__":
    main()
