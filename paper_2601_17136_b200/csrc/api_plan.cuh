// api_plan.cuh -- the host planner of kkm_api.cu (one translation unit with it): everything a
// rank derives from (params, n, d, rank, nranks) -- path, layout, the f1 band pieces / upper-triangle
// units of this rank, splits, and the byte offsets of the caller-owned workspace. Pure host code.
#pragma once

namespace {

thread_local char g_err[1024] = "";

int fail(int code, const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

constexpr double kMaterializeBudget = 160e9;  // bytes of K per rank AUTO will store

int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

// Everything the planner derives from (params, n, d, rank, nranks).
struct Plan {
  int64_t n, d, B, row0, nloc, npad, ldf, dp, ldk, lablen;
  // 1.5D grid: pr x pc, rank = gi + gj * pr. A set = column block gj (output rows
  // of the a2 partials), B set = row block gi (reduction columns). pr = 1: A = own rows, B = all.
  int pr, pc, gi, gj;
  int64_t a0, nA, nApad, b0, nB;
  int k, nranks, rank, max_iter;
  bool materialize, tc, fp16;  // tc: tensor-core a1 (bf16x3 or fp16x3); fp16: fp16x3 split
  int sort_blocks;              // streaming: blocks of the counting sort
  bool spmm_v2;                 // materialised a2 with label-sorted 32-column groups (k <= 64)
  int nsplit, chunks_per_split, nfin, nspmm_pass;
  int64_t rows_per_block;
  size_t kelems;       // materialised K elements (per 16-bit plane)
  int64_t s_rows_pad;  // row pitch of the S (or S partials) finalize reads
  bool need_smine;     // a reduce-scatter delivers S of the own 1D block (Smine)
  // f3 incremental S: moved-point set of at most dmax points
  bool inc;
  bool fused;  // a3 + a4 as one single-CTA kernel (one rank, small n, k <= 16)
  // replicated a3/a4 (1D f1 paths on several ranks): S of ALL points is allreduced (it is summed
  // over the ranks' bands anyway) and every rank runs a3/a4 on all n points -- identical inputs,
  // deterministic kernels, identical labels -- so no c-partial allgather, labels allgather or
  // sizes / changed allreduce remain: one collective per iteration instead of three
  bool repl;
  int64_t a_row0, a_n, a_B;  // the a3/a4 rows: [a_row0, a_row0 + a_n), buffers of a_B rows
  bool a3fix;  // a3 reads the int64 S of spmm_tc directly and finishes c / J in its last block
  int64_t dmax, dpad;
  // f1 symmetric storage (sym.cuh): bands of SYM_TB rows, the rank's share spread by area
  bool sym;
  int T, sym_gmax;
  int64_t sym_items;
  std::vector<SymBand> bands;       // owned bands, ascending I
  std::vector<int32_t> band_desc;   // band -> index into bands, or -1
  bool ssym;                        // f1 on the streaming path (ssym_kernel, ssym.cuh)
  // f4 fp16 K storage (spmm_tc.cuh): the f1 bands in fp16, a2 on the tensor cores
  bool kh;
  int kplanes;                      // 16-bit planes per K value: 1 (FP16) or 2 (FP16X2: hi + lo)
  int ts_nsm;                       // max column splits of a band (informational)
  std::vector<TsBand> tbands;       // owned bands (same order as bands)
  std::vector<TsUnit> tunits;
  int tnl = 16;                     // labels per spmm_tc launch: 16 (k <= 16) or 32 (k <= 32)
  std::vector<TsSlab> tslabs;       // NL = 32: this rank's slabs with column partials, by colstart
  int64_t tcolpart_floats = 0;
  std::vector<int4> units;          // its work units on this rank
  // offsets (bytes) into the workspace
  size_t o_Xf, o_Xhi, o_Xlo, o_norms, o_diag, o_K, o_lab[2], o_sizes[2], o_Spart, o_E,
      o_blockpart, o_rankpart, o_cnorm, o_J, o_changed, o_Dfull, o_bad, o_E2, o_cnorm2, o_rscale,
      o_Shi, o_Slo, o_snorms, o_srscale, o_perm, o_pos, o_seg, o_bcount, o_boff, o_labB, o_Scol, o_Srecv, o_Smine,
      o_codes, o_perm_b, o_groups, o_ngroups, o_bands, o_band_desc, o_colpart, o_colsum, o_work, o_gfirst, o_tmaps, o_tbands, o_tunits, o_tSfix, o_tSint, o_tSmine, o_tcolpart, o_tslabs, o_gregs, o_gmaps, o_a3ctr, o_Sfin, o_units, o_Sfix, o_Sorig, o_Sfmine, o_fxmax, o_Sinc, o_dkey, o_dperm, o_dpos, o_dseg, o_dbc, o_dbo,
      o_Dhi, o_Dlo, o_Dn, o_Dr, o_Sd, o_Sdx, o_Sx, o_mean, o_cmpart, total;
};

int make_plan(const kkm_params *p, int64_t n, int64_t d, int32_t rank, int32_t nranks, Plan *pl) {
  if (!p) return fail(KKM_EINVAL, "params is NULL");
  if (n < 1 || d < 1) return fail(KKM_EINVAL, "n=%lld d=%lld must be >= 1", (long long)n, (long long)d);
  if (nranks < 1 || rank < 0 || rank >= nranks)
    return fail(KKM_EINVAL, "rank %d / nranks %d out of range", rank, nranks);
  if (p->k < 1 || p->k > n) return fail(KKM_EINVAL, "k=%d must satisfy 1 <= k <= n=%lld", p->k, (long long)n);
  if (p->k > KKM_MAX_K) return fail(KKM_EUNSUP, "k=%d > %d clusters is not supported", p->k, KKM_MAX_K);
  if (p->max_iter < 0) return fail(KKM_EINVAL, "max_iter=%d < 0", p->max_iter);
  if (p->kind < 0 || p->kind > 2) return fail(KKM_EINVAL, "unknown kernel kind %d", p->kind);
  if (p->kind == KKM_KERNEL_POLY && (p->degree < 1 || !(p->gamma > 0.0)))
    return fail(KKM_EINVAL, "polynomial kernel needs degree >= 1 and gamma > 0");
  if (p->kind == KKM_KERNEL_GAUSSIAN && !(p->gamma >= 0.0))
    return fail(KKM_EINVAL, "Gaussian kernel needs gamma >= 0");
  if (p->precision != KKM_PREC_BF16X3 && p->precision != KKM_PREC_FP32_SIMT &&
      p->precision != KKM_PREC_FP16X3)
    return fail(KKM_EINVAL, "unknown precision %d", p->precision);
  for (int i = 0; i < 2; ++i)
    if (p->reserved[i]) return fail(KKM_EINVAL, "reserved params must be zero");
  if (p->kstore < KKM_KSTORE_AUTO || p->kstore > KKM_KSTORE_FP16X2)
    return fail(KKM_EINVAL, "unknown kstore %d", p->kstore);
  if (p->incremental != 0 && p->incremental != 1) return fail(KKM_EINVAL, "incremental must be 0 or 1");
  if (p->symmetric != KKM_SYM_AUTO && p->symmetric != KKM_SYM_OFF && p->symmetric != KKM_SYM_ON)
    return fail(KKM_EINVAL, "unknown symmetric mode %d", p->symmetric);
  const int pr = p->grid_rows <= 1 ? 1 : p->grid_rows;
  if (nranks % pr) return fail(KKM_EUNSUP, "grid_rows=%d does not divide nranks=%d", pr, nranks);
  Plan &P = *pl;
  P.n = n;
  P.d = d;
  P.k = p->k;
  P.rank = rank;
  P.nranks = nranks;
  P.max_iter = p->max_iter;
  P.B = ceil_div(n, nranks);
  P.row0 = std::min<int64_t>(n, (int64_t)rank * P.B);
  P.nloc = std::max<int64_t>(0, std::min<int64_t>(P.B, n - P.row0));
  P.npad = P.B * nranks;
  P.pr = pr;
  P.pc = nranks / pr;
  P.gi = rank % pr;
  P.gj = rank / pr;
  P.a0 = std::min<int64_t>(n, (int64_t)P.gj * pr * P.B);
  P.nA = std::max<int64_t>(0, std::min<int64_t>((int64_t)pr * P.B, n - P.a0));
  P.nApad = (int64_t)pr * P.B;
  P.b0 = std::min<int64_t>(n, (int64_t)P.gi * P.pc * P.B);
  P.nB = std::max<int64_t>(0, std::min<int64_t>((int64_t)P.pc * P.B, n - P.b0));
  P.ldf = round_up(d, 4);
  P.dp = round_up(d, TC_BK);  // bf16 operand rows padded to whole 64-element K blocks
  P.ldk = round_up(std::max<int64_t>(P.nB, 1), 32);  // K tile row pitch (columns = B set)
  P.lablen = round_up(std::max(P.npad, round_up(n, 32)), 32);
  P.tc = p->precision == KKM_PREC_BF16X3 || p->precision == KKM_PREC_FP16X3;
  P.fp16 = p->precision == KKM_PREC_FP16X3;
  // f1: symmetric band storage (1D, k <= 16). Bands go to ranks largest first, each to the
  // least-loaded rank (lowest rank on ties): deterministic, area-balanced.
  const bool ssym_elig = p->symmetric != KKM_SYM_OFF && pr == 1;  // streaming f1: any k (ssym.cuh)
  P.kh = p->kstore == KKM_KSTORE_FP16 || p->kstore == KKM_KSTORE_FP16X2;  // AUTO: decided below
  const bool kh_pitch = P.kh || (p->kstore == KKM_KSTORE_AUTO && P.tc);  // the bands if stored are 16-bit
  // materialised f1 bands: fp32 bands (sym.cuh) for k <= 16, 16-bit planes (spmm_tc.cuh) for k <= 32
  const bool sym_elig = p->symmetric != KKM_SYM_OFF && pr == 1 && P.k <= (kh_pitch ? TS_MAX_K : SP_KPMAX);
  P.kplanes = p->kstore == KKM_KSTORE_FP16 ? 1 : 2;
  const bool sym_ok = sym_elig && (p->symmetric == KKM_SYM_ON || P.kh || n >= 8 * SYM_TB);
  double kbytes = (double)P.nApad * (double)P.ldk * 4.0;
  P.T = (int)ceil_div(n, SYM_TB);
  P.sym_gmax = sym_gmax(P.k);
  P.bands.clear();
  P.band_desc.assign(P.T, -1);
  P.sym_items = 0;
  if (sym_ok) {
    std::vector<double> load(nranks, 0.0);
    int64_t koff = 0, cpoff = 0, csoff = 0;
    for (int I = 0; I < P.T; ++I) {
      const int64_t rows = std::min<int64_t>(SYM_TB, n - (int64_t)I * SYM_TB);
      // 16-bit planes (spmm_tc): rows padded to 128 elements = 256 B, so each 128-column chunk
      // of a row is one 256-B aligned L2 promotion unit (no re-fetch of a neighbour's bytes)
      const int64_t ldb = round_up(n - (int64_t)I * SYM_TB, kh_pitch ? 128 : 32);
      int owner = 0;
      for (int r = 1; r < nranks; ++r)
        if (load[r] < load[owner]) owner = r;
      load[owner] += (double)rows * (double)ldb;
      if (owner != rank) continue;
      SymBand b;
      b.band = I;
      b.row0 = 0;
      b.rows = (int32_t)rows;
      b.ldb = (int32_t)ldb;
      b.koff = koff;
      b.cpoff = cpoff;
      b.csoff = csoff;
      const int64_t chunks = ceil_div(ldb, SYM_CH);  // spmm_sym chunk width
      b.nsplit = (int32_t)ceil_div(chunks, SP_MAX_CHUNKS_PER_SPLIT * 1024 / SYM_CH);  // <= ~1024 fp32 terms per lane
      b.cps = (int32_t)ceil_div(chunks, b.nsplit);
      b.item0 = P.sym_items;
      P.sym_items += (int64_t)P.sym_gmax * b.nsplit;
      koff += rows * ldb;
      cpoff += (int64_t)P.sym_gmax * std::max<int64_t>(0, ldb - SYM_TB);
      csoff += (int64_t)P.k * std::max<int64_t>(0, ldb - SYM_TB);
      P.band_desc[I] = (int32_t)P.bands.size();
      P.bands.push_back(b);
    }
    kbytes = (double)koff * (P.kh ? 2.0 * P.kplanes : 4.0);
  }
  if (p->path == KKM_PATH_MATERIALIZE) {
    P.materialize = true;
  } else if (p->path == KKM_PATH_STREAM) {
    P.materialize = false;
  } else if (p->path == KKM_PATH_AUTO) {
    P.materialize = kbytes <= kMaterializeBudget;
  } else {
    return fail(KKM_EINVAL, "unknown path %d", p->path);
  }
  if (!P.materialize) {
    if (!P.tc)
      return fail(KKM_EUNSUP, "the streaming path needs a tensor-core precision (FP16X3 or BF16X3)");
  }
  // AUTO: the hi + lo fp16 planes (fp32-class, a2 on the tensor cores) whenever the bands are stored
  if (p->kstore == KKM_KSTORE_AUTO && P.materialize && sym_ok && P.tc) P.kh = true;
  if (P.kh && !(P.materialize && sym_ok && P.tc))
    return fail(KKM_EUNSUP, "16-bit K storage needs a tensor-core precision and the materialised f1 bands "
                            "(1D, k <= 32, symmetric != OFF)");
  // v1 (one-hot FFMA2) is faster for k <= 16 (5.4 TB/s at k = 10); v2 (sorted groups, shuffle
  // bound at ~3.9 TB/s for any k) replaces v1's ceil(k/16) passes over K for 16 < k <= 64.
  P.spmm_v2 = P.k > SP_KPMAX && P.k <= SG_MAX_K;
  if (P.materialize && P.spmm_v2) {
    const int64_t nchunks = ceil_div(P.ldk, SG_CH);
    const int64_t groups = ceil_div(std::max<int64_t>(P.nA, 1), SG_ROWS);
    // splits: bound the chunks per item, and give >= ~4 items per SM for load balance
    int64_t ns = std::max<int64_t>(ceil_div(nchunks, SG_MAX_CHUNKS_PER_SPLIT), ceil_div(4 * 148, groups));
    ns = std::min<int64_t>(std::max<int64_t>(ns, 1), nchunks);
    P.nsplit = (int)ns;
    P.chunks_per_split = (int)ceil_div(nchunks, P.nsplit);
  } else if (P.materialize) {
    const int ch = 2048;  // chunk width of the one-hot kernel (spmm.cuh SpRows::CH)
    const int64_t nchunks = ceil_div(P.ldk, ch);
    P.nsplit = (int)ceil_div(nchunks, SP_MAX_CHUNKS_PER_SPLIT * 1024 / ch);
    P.chunks_per_split = (int)ceil_div(nchunks, P.nsplit);
  } else {
    // the fused streaming kernel takes units of W column tiles in G-row supertiles dynamically
    // (tc3.cuh T2StreamSched); it sums S in int64 fixed point (one [rows][k] array), converted
    // once to fp64: one partial for a3 (nsplit = 1).
    P.nsplit = 1;
    P.chunks_per_split = 0;
  }
  P.sym = P.materialize && sym_ok;
  // f1 on the streaming path: upper-triangle pair tiles of the label-sorted K as work units
  // (row tile, first column tile, count), in an L2-friendly order; each rank takes a contiguous
  // run of that order holding ~1/P of the tiles, and its pairs take the run's units dynamically
  // (ssym.cuh), so the units in flight on a GPU stay consecutive in the order
  P.ssym = !P.materialize && ssym_elig && P.tc;
  P.units.clear();
  if (P.ssym) {
    const int64_t Tt = ceil_div(n, 256);
    std::vector<int4> all;
    // Default: a G x G supertile raster -- patches of G row tiles x G column tiles of the upper
    // triangle, patch row by patch row, inside a patch W column tiles at a time across its G row
    // tiles; a unit = (row tile, W column tiles). The ~74 units in flight cover ~G row tiles x a
    // few W-groups of columns: ~30 MB of split operands in L2, each B tile read by G units in a
    // row. Measured at n = 1M (dynamic schedule): G x W = 32 x 16 1.50-1.52 s, DRAM 258 GB, L2 hit
    // 94 %; 16 x 4 1.56 s; the block-major order (G = 0: units = (row tile, aligned block of BS
    // column tiles), block by block) 1.55 s, DRAM 959 GB. KKM_SSYM_G / _W / _BS: A/B runs.
    int64_t G = 32, W = 16, BS = 16;
    if (const char *e = std::getenv("KKM_SSYM_G")) G = std::max<int64_t>(0, std::atoll(e));
    if (const char *e = std::getenv("KKM_SSYM_W")) W = std::max<int64_t>(1, std::atoll(e));
    if (const char *e = std::getenv("KKM_SSYM_BS")) BS = std::max<int64_t>(1, std::atoll(e));
    if (G > 0) {
      for (int64_t I = 0; I * G < Tt; ++I)
        for (int64_t J = I; J * G < Tt; ++J) {
          const int64_t je = std::min(Tt, (J + 1) * G);
          for (int64_t t0 = J * G; t0 < je; t0 += W)
            for (int64_t tm = I * G; tm < std::min(Tt, (I + 1) * G); ++tm) {
              const int64_t a = std::max(tm, t0), e = std::min(je, t0 + W);
              if (a < e) all.push_back(make_int4((int)tm, (int)a, (int)(e - a), 0));
            }
        }
    } else {
      for (int64_t b = 0; b * BS < Tt; ++b)
        for (int64_t tm = 0; tm < std::min(Tt, (b + 1) * BS); ++tm) {
          const int64_t a = std::max(tm, b * BS), e = std::min(Tt, (b + 1) * BS);
          all.push_back(make_int4((int)tm, (int)a, (int)(e - a), 0));
        }
    }
    // contiguous runs by cumulative tile count: rank r takes the units whose first tile falls in
    // [r total / P, (r + 1) total / P) of the running count (imbalance <= one unit)
    int64_t total = 0;
    for (const int4 &u : all) total += u.z;
    int64_t cum = 0;
    for (const int4 &u : all) {
      const int64_t owner = std::min<int64_t>(nranks - 1, cum * nranks / std::max<int64_t>(total, 1));
      if (owner == rank) P.units.push_back(u);
      cum += u.z;
    }
    P.nsplit = 1;
  }
  P.tbands.clear();
  P.tunits.clear();
  P.ts_nsm = 0;
  if (P.sym && P.kh && nranks > 1) {
    // 16-bit bands on several ranks: spread 512-row pieces of the bands by area (finer than whole
    // bands, so the ranks' a2 work is balanced to ~1 % instead of ~10 %)
    P.bands.clear();
    P.band_desc.assign(P.T, -1);  // (used by the fp32 band path only)
    std::vector<double> load(nranks, 0.0);
    int64_t koff = 0;
    constexpr int PIECE = TS_SLAB_TILES * TS_ROWS;
    for (int I = 0; I < P.T; ++I)
      for (int r0 = 0; r0 < SYM_TB && (int64_t)I * SYM_TB + r0 < n; r0 += PIECE) {
        const int64_t rows = std::min<int64_t>(PIECE, n - (int64_t)I * SYM_TB - r0);
        const int64_t ldb = round_up(n - (int64_t)I * SYM_TB, 128);
        int owner = 0;
        for (int r = 1; r < nranks; ++r)
          if (load[r] < load[owner]) owner = r;
        load[owner] += (double)rows * (double)ldb;
        if (owner != rank) continue;
        SymBand b{};
        b.band = I;
        b.row0 = r0;
        b.rows = (int32_t)rows;
        b.ldb = (int32_t)ldb;
        b.koff = koff;
        koff += rows * ldb;
        P.bands.push_back(b);
      }
  }
  if (P.sym && P.kh) {  // f4: units = (piece, 512-row slab, <= split chunks of 128 columns)
    // split: 16 chunks, or 8 when that leaves fewer than ~32 units per SM (the last wave of 4 MB
    // units idled SMs at config 2 on 4 GPUs; at config 3 the smaller units cost ~6 %)
    int64_t cslabs = 0;
    for (const SymBand &sb : P.bands)
      cslabs += ceil_div(sb.rows, TS_SLAB_TILES * TS_ROWS) * ceil_div(sb.ldb, TS_CH);
    const int split = cslabs / 16 >= 32 * 148 ? 16 : 8;
    P.tnl = P.k <= 16 ? 16 : 32;
    P.tslabs.clear();
    int64_t cpoff = 0;  // NL = 32: the slabs' column partials [slab][NL][ldb - TB]
    for (size_t b = 0; b < P.bands.size(); ++b) {
      const SymBand &sb = P.bands[b];
      TsBand t;
      t.koff = sb.koff;
      t.cpoff = cpoff;
      t.band = sb.band;
      t.row0 = sb.row0;
      t.ldb = sb.ldb;
      t.rows = sb.rows;
      const int nchunks = (int)ceil_div(t.ldb, TS_CH);
      t.nsplit = (int)ceil_div(nchunks, split);
      const int slabs = (int)ceil_div(t.rows, TS_SLAB_TILES * TS_ROWS);
      P.ts_nsm = std::max(P.ts_nsm, t.nsplit);
      for (int sl = 0; sl < slabs; ++sl)
        for (int sp = 0; sp < t.nsplit; ++sp)
          P.tunits.push_back(TsUnit{(int32_t)b, sl, sp * split, std::min(split, nchunks - sp * split)});
      P.tbands.push_back(t);
      const int64_t w = std::max<int64_t>(0, (int64_t)t.ldb - SYM_TB);
      if (P.tnl == 32 && w > 0)
        for (int sl = 0; sl < slabs; ++sl) {
          P.tslabs.push_back(TsSlab{(int64_t)(t.band + 1) * SYM_TB, w, cpoff + (int64_t)sl * P.tnl * w});
        }
      if (P.tnl == 32) cpoff += (int64_t)slabs * P.tnl * w;
    }
    std::stable_sort(P.tslabs.begin(), P.tslabs.end(),
                     [](const TsSlab &x, const TsSlab &y) { return x.colstart < y.colstart; });
    P.tcolpart_floats = cpoff;
  }
  if (P.sym) {  // S partials over all rows (owned bands lie anywhere)
    P.nApad = P.npad;
    P.nsplit = 1;
    for (const SymBand &b : P.bands) P.nsplit = std::max(P.nsplit, (int)b.nsplit);
    if (P.kh) P.nsplit = 1;  // (Spart unused: spmm_tc sums S in int64 fixed point)
    P.chunks_per_split = 0;
  } else {
    P.bands.clear();
    P.band_desc.clear();
  }
  if (P.ssym) P.nApad = P.npad;
  P.s_rows_pad = (P.pr > 1 || ((P.sym || P.ssym) && P.nranks > 1)) ? P.B : P.nApad;  // == need_smine
  P.inc = p->incremental == 1;
  P.repl = nranks > 1 && P.pr == 1 && (P.sym || P.ssym) && !P.inc;
  P.a_row0 = P.repl ? 0 : P.row0;
  P.a_n = P.repl ? n : P.nloc;
  P.a_B = P.repl ? P.npad : P.B;
  if (P.repl) P.s_rows_pad = P.npad;
  P.fused = (nranks == 1 || P.repl) && n <= FUSED_MAX_ROWS && P.k <= 16;
  P.a3fix = P.kh && P.sym && !P.inc && !P.fused && (nranks == 1 || P.repl);
  if (P.inc && (P.pr > 1 || !P.tc))
    return fail(KKM_EUNSUP, "incremental S needs the 1D algorithm and a tensor-core precision");
  P.dmax = std::max<int64_t>(1, n / 16);
  P.dpad = round_up(P.dmax, 256);
  P.sort_blocks = (int)ceil_div(std::max<int64_t>(P.nB, 1), SORT_BLOCK);
  P.nspmm_pass = (int)ceil_div(P.k, SP_KPMAX);
  P.nfin = (int)std::min<int64_t>(1024, ceil_div(std::max<int64_t>(P.a_n, 1), FIN_THREADS));
  P.rows_per_block = ceil_div(std::max<int64_t>(P.a_n, 1), P.nfin);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += (bytes + 255) / 256 * 256;
    return o;
  };
  const int64_t k1 = P.k + 1;
  P.o_Xf = take((size_t)P.npad * P.ldf * 4);
  P.o_mean = take((size_t)P.ldf * 4);
  P.o_cmpart = p->kind == KKM_KERNEL_GAUSSIAN ? take((size_t)ceil_div(n, CM_ROWS) * P.ldf * 8) : 0;
  P.o_Xhi = P.tc ? take((size_t)P.npad * P.dp * 2) : 0;
  P.o_Xlo = P.tc ? take((size_t)P.npad * P.dp * 2) : 0;
  P.o_rscale = take((size_t)P.npad * 4);
  P.o_norms = take((size_t)P.npad * 4);
  P.o_diag = take((size_t)P.a_B * 8);
  size_t kfloats = (size_t)P.nApad * P.ldk;
  size_t cpfloats = 0, csdoubles = 0;
  if (P.sym) {
    kfloats = 0;
    for (const SymBand &b : P.bands) {
      kfloats += (size_t)b.rows * b.ldb;
      cpfloats += (size_t)P.sym_gmax * std::max<int64_t>(0, b.ldb - SYM_TB);
      csdoubles += (size_t)P.k * std::max<int64_t>(0, b.ldb - SYM_TB);
    }
  }
  P.o_K = P.materialize ? take(std::max<size_t>(kfloats, 1) * (P.kh ? 2 * P.kplanes : 4)) : 0;
  P.kelems = kfloats;  // elements per plane
  P.o_lab[0] = take((size_t)P.lablen * 4);
  P.o_lab[1] = take((size_t)P.lablen * 4);
  P.o_sizes[0] = take((size_t)P.k * 4);
  P.o_sizes[1] = take((size_t)P.k * 4);
  P.o_Spart = take((size_t)P.nsplit * P.nApad * P.k * 8);
  P.o_E = take((size_t)P.a_B * P.k * 8);
  P.o_blockpart = take((size_t)P.nfin * k1 * 8);
  P.o_rankpart = take((size_t)nranks * k1 * 8);
  P.o_cnorm = take((size_t)P.k * 8);
  P.o_J = take((size_t)(P.max_iter + 2) * 8);
  P.o_changed = take((size_t)(P.max_iter + 2) * 8);
  P.o_Dfull = take((size_t)P.a_B * P.k * 8);
  P.o_bad = take(16);
  P.o_E2 = take((size_t)P.a_B * P.k * 8);
  P.o_cnorm2 = take((size_t)P.k * 8);
  if (!P.materialize) {
    P.o_Shi = take((size_t)P.npad * P.dp * 2);
    P.o_Slo = take((size_t)P.npad * P.dp * 2);
    P.o_snorms = take((size_t)P.npad * 4);
    P.o_srscale = take((size_t)P.npad * 4);
    P.o_perm = take((size_t)P.lablen * 4);
    P.o_pos = take((size_t)P.lablen * 4);
    P.o_seg = take((size_t)(P.k + 1) * 4);
    P.o_bcount = take((size_t)P.sort_blocks * P.k * 4);
    P.o_boff = take((size_t)P.sort_blocks * P.k * 4);
    if (!P.ssym) P.o_Sx = take((size_t)P.nApad * P.k * 8);  // the full streaming kernel's int64 S
  }
  if (P.materialize && P.spmm_v2) P.o_codes = take((size_t)P.ldk * 4);
  if (P.pr > 1) {
    P.o_labB = take((size_t)P.ldk * 4);
    P.o_Scol = take((size_t)P.nApad * P.k * 8);
    P.o_Srecv = take((size_t)P.nApad * P.k * 8);  // the column peers' pieces (slot = their row rank)
  }
  P.need_smine = P.pr > 1 || ((P.sym || P.ssym) && P.nranks > 1 && !P.repl);  // S of the own block after a reduce-scatter
  if (P.need_smine) P.o_Smine = take((size_t)P.B * P.k * 8);
  if (P.ssym) {
    P.o_units = take(std::max<size_t>(P.units.size(), 1) * sizeof(int4));
    P.o_Sfix = take((size_t)P.npad * P.k * 8);
    P.o_Sorig = P.nranks > 1 ? take((size_t)P.npad * P.k * 8) : 0;
    P.o_Sfmine = P.nranks > 1 ? take((size_t)P.B * P.k * 8) : 0;
  }
  if (P.inc) {
    const int64_t nblk = ceil_div(P.n, SORT_BLOCK);
    P.o_Sinc = take((size_t)P.B * P.k * 8);
    P.o_dkey = take((size_t)P.lablen * 4);
    P.o_dperm = take((size_t)P.lablen * 4);
    P.o_dpos = take((size_t)P.lablen * 4);
    P.o_dseg = take((size_t)(P.k + 2) * 4);
    P.o_dbc = take((size_t)nblk * (P.k + 1) * 4);
    P.o_dbo = take((size_t)nblk * (P.k + 1) * 4);
    P.o_Dhi = take((size_t)P.dpad * P.dp * 2);
    P.o_Dlo = take((size_t)P.dpad * P.dp * 2);
    P.o_Dn = take((size_t)P.dpad * 4);
    P.o_Dr = take((size_t)P.dpad * 4);
    P.o_Sd = take((size_t)P.B * P.k * 8);   // fp64 S of the moved points' pass
    P.o_Sdx = take((size_t)P.B * P.k * 8);  // its int64 fixed-point sums
  }
  if (P.sym || P.ssym) P.o_work = take(4 * 4);  // item schedulers: [0, 2) spmm_tc, [2, 4) ssym (zero between launches)
  if (P.sym) {
    P.o_perm_b = take((size_t)P.T * SYM_TB * 4);
    P.o_groups = take((size_t)P.T * P.sym_gmax * sizeof(SymGroup));
    P.o_ngroups = take((size_t)P.T * 4);
    P.o_bands = take(std::max<size_t>(P.bands.size(), 1) * sizeof(SymBand));
    P.o_band_desc = take((size_t)P.T * 4);
    P.o_colpart = take(P.kh ? 4 : std::max<size_t>(cpfloats, 1) * 4);
    P.o_colsum = take(P.kh ? 8 : std::max<size_t>(csdoubles, 1) * 8);
    P.o_gfirst = take((size_t)P.T * (P.k + 1) * 4);
    P.o_Sfin = take((size_t)P.npad * P.k * 8);
    if (P.tc) {  // one GEMM launch over all owned band pieces: regions + output maps
      P.o_gregs = take(std::max<size_t>(P.bands.size(), 1) * sizeof(T2Region));
      P.o_gmaps = take(std::max<size_t>(P.bands.size() * (P.kh ? P.kplanes : 1), 1) * sizeof(CUtensorMap));
    }
  }
  if (P.sym && P.kh) {
    P.o_tmaps = take(std::max<size_t>(P.tbands.size() * P.kplanes, 1) * sizeof(CUtensorMap));
    P.o_tbands = take(std::max<size_t>(P.tbands.size(), 1) * sizeof(TsBand));
    P.o_tunits = take(std::max<size_t>(P.tunits.size(), 1) * sizeof(TsUnit));
    P.o_tSfix = take((size_t)P.npad * P.k * 8);  // int64 fixed-point S, [label][row]
    P.o_tSint = P.nranks > 1 ? take((size_t)P.npad * P.k * 8) : 0;
    P.o_tSmine = P.nranks > 1 ? take((size_t)P.B * P.k * 8) : 0;
    if (P.tnl == 32) {
      P.o_tcolpart = take((size_t)std::max<int64_t>(P.tcolpart_floats, 1) * 4);
      P.o_tslabs = take(std::max<size_t>(P.tslabs.size(), 1) * sizeof(TsSlab));
    }
  }
  P.o_a3ctr = take(16);
  P.o_fxmax = take(16);
  P.total = off;
  return KKM_OK;
}

}  // namespace
