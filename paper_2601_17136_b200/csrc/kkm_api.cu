// kkm_api.cu -- the C-ABI of include/kkm.h: handle, workspace planner, one-time setup,
// the clustering loop of Alg. 1 over the kernels in *.cuh, the NCCL
// exchange steps of the 1D algorithm, and the test hooks.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <chrono>
#include <thread>
#include <vector>

#include "kkm.h"
#include "common.cuh"
#include "gemm_simt.cuh"
#include "gemm_tc.cuh"
#include "kpp.cuh"
#include "prep.cuh"
#include "sort.cuh"
#include "spmm.cuh"
#include "stream.cuh"
#include "spmm_tc.cuh"
#include "sym.cuh"
#include "tc2.cuh"
#include "ssym.cuh"
#include "tc3.cuh"
#include "update.cuh"

using namespace kkm;

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
  int stream_splits = 1;  // column splits per row tile of the full streaming kernel (tc3_stream_kernel)
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
  std::vector<int4> units;          // its work units on this rank
  // offsets (bytes) into the workspace
  size_t o_Xf, o_Xhi, o_Xlo, o_norms, o_diag, o_K, o_lab[2], o_sizes[2], o_Spart, o_E,
      o_blockpart, o_rankpart, o_cnorm, o_J, o_changed, o_Dfull, o_bad, o_E2, o_cnorm2, o_rscale,
      o_Shi, o_Slo, o_snorms, o_srscale, o_perm, o_pos, o_seg, o_bcount, o_boff, o_labB, o_Scol, o_Smine,
      o_codes, o_perm_b, o_groups, o_ngroups, o_bands, o_band_desc, o_colpart, o_colsum, o_work, o_gfirst, o_tmaps, o_tbands, o_tunits, o_tSfix, o_tSint, o_tSmine, o_gregs, o_gmaps, o_a3ctr, o_Sfin, o_units, o_Sfix, o_Sorig, o_Sfmine, o_fxmax, o_Sinc, o_dkey, o_dperm, o_dpos, o_dseg, o_dbc, o_dbo,
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
  const bool sym_elig = p->symmetric != KKM_SYM_OFF && pr == 1 && P.k <= SP_KPMAX;
  const bool ssym_elig = p->symmetric != KKM_SYM_OFF && pr == 1;  // streaming f1: any k (ssym.cuh)
  P.kh = p->kstore == KKM_KSTORE_FP16 || p->kstore == KKM_KSTORE_FP16X2;  // AUTO: decided below
  const bool kh_pitch = P.kh || (p->kstore == KKM_KSTORE_AUTO && P.tc);  // the bands if stored are 16-bit
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
                            "(1D, k <= 16, symmetric != OFF)");
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
    // work units of the fused kernel = 128-row tiles x column splits; 148 SMs assumed for the
    // load-balance choice (B200). Work units = 256-row pair tiles x column splits (74 CTA pairs),
    // ordered tile-major (the clusters working on one row tile's splits share its A operand in
    // L2). Splits: at most 512 256-column tiles per unit, which bounds how far the concurrent
    // sweeps over B drift apart (measured at n = 1M: 4.41 -> 3.92 s per iteration); then the best
    // last-wave fill. The kernel sums S in int64 fixed point (one [rows][k] array, any number of
    // splits), converted once to fp64: one partial for a3 (nsplit = 1).
    const int64_t tiles_n = ceil_div(std::max<int64_t>(P.nB, 1), 256);
    const int64_t s_l2 = ceil_div(tiles_n, 512);
    const int s_bal = ts_choose_splits((P.nA + 1) / 2, P.nB, 74);
    P.stream_splits = (int)std::max<int64_t>(s_l2, s_bal);
    P.nsplit = 1;
    P.chunks_per_split = 0;
  }
  P.sym = P.materialize && sym_ok;
  // f1 on the streaming path: upper-triangle pair tiles of the label-sorted K, work units
  // (row tile, first column tile, count) of <= 512 tiles, spread over the ranks largest first
  P.ssym = !P.materialize && ssym_elig && P.tc;
  P.units.clear();
  if (P.ssym) {
    const int64_t Tt = ceil_div(n, 256);
    std::vector<int4> all;
    // units = (row tile, globally aligned block of <= BS column tiles); a rank's units run
    // block-major (below), so the ~74 pairs running at once sweep the same block of B tiles
    // with different row tiles: the block (BS x 256 rows of the split operand) and the pairs'
    // A tiles stay L2-resident
    int64_t BS = 32;
    if (const char *e = std::getenv("KKM_SSYM_BS")) BS = std::max<int64_t>(1, std::atoll(e));
    const bool tile_major = std::getenv("KKM_SSYM_TILE_MAJOR") != nullptr;  // (the round-1 order, A/B only)
    // G > 0: single-tile units in a supertile raster -- G x G patches of the upper triangle, patch
    // by patch, each patch column by column -- so the ~74 tiles in flight cover a compact patch
    // (~9 row tiles x ~9 column tiles: ~15 MB of operands in L2 instead of 74 row tiles + a block)
    int64_t G = 0;
    if (const char *e = std::getenv("KKM_SSYM_G")) G = std::max<int64_t>(0, std::atoll(e));
    if (G > 0) {
      for (int64_t I = 0; I * G < Tt; ++I)
        for (int64_t J = I; J * G < Tt; ++J)
          for (int64_t tn = J * G; tn < std::min(Tt, (J + 1) * G); ++tn)
            for (int64_t tm = I * G; tm < std::min(Tt, (I + 1) * G) && tm <= tn; ++tm)
              all.push_back(make_int4((int)tm, (int)tn, 1, 0));
    } else {
      for (int64_t tm = 0; tm < Tt; ++tm)
        for (int64_t b = tm / BS; b * BS < Tt; ++b) {
          const int64_t a = std::max(tm, b * BS), e = std::min(Tt, (b + 1) * BS);
          all.push_back(make_int4((int)tm, (int)a, (int)(e - a), 0));
        }
    }
    std::vector<int64_t> load(nranks, 0);
    std::vector<int> order(all.size());
    for (size_t i = 0; i < all.size(); ++i) order[i] = (int)i;
    std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return all[x].z > all[y].z; });
    std::vector<char> mine(all.size(), 0);
    for (int i : order) {
      int r = 0;
      for (int q = 1; q < nranks; ++q)
        if (load[q] < load[r]) r = q;
      load[r] += all[i].z;
      if (r == rank) mine[i] = 1;
    }
    for (size_t i = 0; i < all.size(); ++i)
      if (mine[i]) P.units.push_back(all[i]);
    if (!tile_major && G == 0)  // block-major order on the rank: (column block, row tile)
      std::stable_sort(P.units.begin(), P.units.end(), [&](const int4 &x, const int4 &y) {
        const int64_t bx = x.y / BS, by = y.y / BS;
        return bx != by ? bx < by : x.x < y.x;
      });
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
    for (size_t b = 0; b < P.bands.size(); ++b) {
      const SymBand &sb = P.bands[b];
      TsBand t;
      t.koff = sb.koff;
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
    }
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
  if (P.sym) {
    P.o_perm_b = take((size_t)P.T * SYM_TB * 4);
    P.o_groups = take((size_t)P.T * P.sym_gmax * sizeof(SymGroup));
    P.o_ngroups = take((size_t)P.T * 4);
    P.o_bands = take(std::max<size_t>(P.bands.size(), 1) * sizeof(SymBand));
    P.o_band_desc = take((size_t)P.T * 4);
    P.o_colpart = take(P.kh ? 4 : std::max<size_t>(cpfloats, 1) * 4);
    P.o_colsum = take(P.kh ? 8 : std::max<size_t>(csdoubles, 1) * 8);
    P.o_work = take(2 * 4);  // spmm_sym's item scheduler
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
  }
  P.o_a3ctr = take(16);
  P.o_fxmax = take(16);
  P.total = off;
  return KKM_OK;
}

}  // namespace

// CUDA events owned for one scope (destroyed on every exit path, errors included).
struct EventList {
  std::vector<cudaEvent_t> v;
  EventList() = default;
  EventList(const EventList &) = delete;
  EventList &operator=(const EventList &) = delete;
  ~EventList() { clear(); }
  void clear() {
    for (cudaEvent_t e : v) cudaEventDestroy(e);
    v.clear();
  }
  // creates and records one event; false if the runtime refused
  bool record(cudaStream_t st) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return false;
    v.push_back(e);
    return cudaEventRecord(e, st) == cudaSuccess;
  }
};

// Label-sorted copy of a point set (the B operand of the streaming kernel) and its sort.
struct SortedSet {
  uint16_t *hi, *lo;
  float *norms, *rscale;
  int32_t *perm, *pos, *seg, *bcount, *boff;
};

struct kkm_ctx {
  kkm_params p;
  Plan P;
  cudaStream_t st = nullptr;
  ncclComm_t comm = nullptr;
  int num_sms = 148;
  uint8_t *ws = nullptr;
  float *Xf = nullptr, *norms = nullptr, *K = nullptr;
  float *mean = nullptr;  // Gaussian: the column means X was centered on (0 otherwise)
  uint16_t *Xhi = nullptr, *Xlo = nullptr;  // bf16 or fp16 split of X (P.tc)
  float *rscale = nullptr;                   // 1 / s_i of the fp16 split
  double *diag, *Spart, *E, *blockpart, *rankpart, *cnorm, *J, *Dfull;
  double *E2, *cnorm2;  // E / c of the final-labels pass (kept apart from the last iteration's)
  // streaming path: cluster-sorted operands and the sort
  uint16_t *Shi = nullptr, *Slo = nullptr;
  float *snorms = nullptr, *srscale = nullptr;
  int32_t *perm = nullptr, *pos = nullptr, *seg = nullptr, *bcount = nullptr, *boff = nullptr;
  TcStream ts, ts_predict;  // tensor maps of the clustering loop / of kkm_predict
  // 1.5D: padded labels of the B set, column-block partials, own-block sums; column comm
  int32_t *labB = nullptr;
  double *Scol = nullptr, *Smine = nullptr;
  uint32_t *codes = nullptr;  // SpMM v2 per-iteration group codes
  // f1 symmetric storage
  int32_t *perm_b = nullptr, *ngroups = nullptr, *band_desc = nullptr, *gfirst = nullptr;
  SymGroup *groups = nullptr;
  SymBand *bands = nullptr;
  float *colpart = nullptr;
  double *colsum = nullptr, *Sfin = nullptr;
  int32_t *work = nullptr;  // spmm_sym's item scheduler (2 counters, zero between launches)
  unsigned *a3ctr = nullptr;  // finalize's last-block counter (zero between launches)
  // peer-memory exchange of S (16-bit bands, replicated a3, several ranks): own IPC buffer
  // [2 epochs][k][npad] int64 + flag + peer table; peers' buffers mapped with cudaIpcOpenMemHandle
  bool p2p = false;
  uint8_t *xbuf = nullptr;
  std::vector<void *> xpeers;  // opened peer mappings (closed in destroy)
  const uint8_t **xtable = nullptr;  // device [nranks] bases (inside xbuf)
  size_t xflag_off = 0;              // byte offset of the epoch flag in every exchange buffer
                                     // (+64: this rank's timed-out word, checked by check_p2p)
  unsigned long long epoch = 0;
  unsigned long long p2p_timeout_ns = 0;
  // f4 fp16 K storage
  CUtensorMap *tmaps = nullptr;
  TsBand *tbands = nullptr;
  TsUnit *tunits = nullptr;
  long long *tSfix = nullptr, *tSint = nullptr, *tSmine = nullptr;
  float kscale = 1.f;  // stored K = K * kscale (a power of two)
  double tfxm = 1.0, tfx_inv = 1.0;  // S fixed point: drained (scaled) sums x tfxm; back x tfx_inv
  // f1 streaming: units, int64 fixed-point S (sorted order), its original-order copy
  int4 *units = nullptr;
  long long *Sfix = nullptr, *Sorig = nullptr, *Sfmine = nullptr;
  float *fxmax = nullptr;
  double fx_scale = 1.0, fx_inv = 1.0;
  // f3 incremental S
  double *Sinc = nullptr, *Sd = nullptr;
  long long *Sdx = nullptr;
  int32_t *dkey = nullptr;
  SortedSet dset{};
  bool s_valid = false;  // Sinc holds S of the current labels
  TcStream ts_delta;
  ncclComm_t colcomm = nullptr;
  int32_t *lab[2], *sizes[2];
  unsigned long long *changed;
  int *bad;
  int cur = 0;  // labels[cur] / sizes[cur] are the labels entering the next iteration
  bool poisoned = false;
  int chain_kb = 0;      // K-blocks per accumulation chain of every tensor-core kernel (0: CH_CKB; KKM_CHAIN_KB)
  bool have_last = false;
  bool cnorm2_valid = false;  // cnorm2 holds c of the current labels (after kkm_fit / kkm_objective)
  int64_t launches = 0;
  float phase_ms[KKM_NPHASES] = {0, 0, 0, 0, 0, 0};
  bool time_a2 = false;             // timing mode, inside the kkm_fit loop
  EventList a2ev;                   // (start, end) pairs around the dominant a2 kernel
  KappaParams kp;
  TcGemm tc;
};

namespace {

#define CK(call)                                                                         \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess) {                                                             \
      h->poisoned = true;                                                                \
      return fail(KKM_ECUDA, "%s:%d %s: %s", __FILE__, __LINE__, #call, cudaGetErrorString(e_)); \
    }                                                                                    \
  } while (0)

#define CKL()                                                                            \
  do {                                                                                   \
    ++h->launches;                                                                       \
    cudaError_t e_ = cudaGetLastError();                                                 \
    if (e_ != cudaSuccess) {                                                             \
      h->poisoned = true;                                                                \
      return fail(KKM_ECUDA, "%s:%d launch: %s", __FILE__, __LINE__, cudaGetErrorString(e_)); \
    }                                                                                    \
  } while (0)

#define CKN(call)                                                                        \
  do {                                                                                   \
    ncclResult_t r_ = (call);                                                            \
    if (r_ != ncclSuccess) {                                                             \
      h->poisoned = true;                                                                \
      return fail(KKM_ENCCL, "%s:%d %s: %s", __FILE__, __LINE__, #call, ncclGetErrorString(r_)); \
    }                                                                                    \
  } while (0)

#define CKR(expr)        \
  do {                   \
    int rc_ = (expr);    \
    if (rc_) return rc_; \
  } while (0)

// Brackets the dominant a2 kernel launch(es) with CUDA events (timing mode, kkm_fit loop).
void a2_mark(kkm_ctx *h) {
  if (h->time_a2) h->a2ev.record(h->st);
}

// Host or device pointer copy on the handle's stream.
int copy_any(kkm_ctx *h, void *dst, const void *src, size_t bytes) {
  CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, h->st));
  return KKM_OK;
}

template <int KP>
int launch_spmm_kp(kkm_ctx *h, const int32_t *labels, int c0) {
  const Plan &P = h->P;
  CK(ensure_smem_attr((const void *)spmm_onehot_kernel<KP>, spmm_smem_bytes<KP>()));
  const int64_t items = ceil_div(P.nA, SpRows<KP>::R) * P.nsplit;
  const int grid = (int)std::min<int64_t>(items, h->num_sms);
  spmm_onehot_kernel<KP><<<grid, SpRows<KP>::THREADS, spmm_smem_bytes<KP>(), h->st>>>(
      h->K, P.ldk, P.nA, labels, P.k, c0, P.nsplit, P.chunks_per_split, P.nApad, h->Spart);
  CKL();
  return KKM_OK;
}

// Sorts the points [b0, b0 + nB) of the handle's X by label (stable counting sort) and gathers
// their split operands, norms and scales in that order into o (rows [nB, rows) zeroed).
int sort_gather(kkm_ctx *h, const int32_t *labB, int64_t b0, int64_t nB, int64_t rows, const SortedSet &o) {
  const Plan &P = h->P;
  const int k = P.k;
  const int nblk = (int)ceil_div(std::max<int64_t>(nB, 1), SORT_BLOCK);
  sort_count_kernel<<<nblk, 256, (size_t)k * 4, h->st>>>(labB, nB, k, o.bcount);
  CKL();
  sort_scan_kernel<<<k + 1, 1024, 1024 * 4, h->st>>>(o.bcount, nblk, k, o.boff, o.seg);
  CKL();
  sort_scatter_kernel<<<nblk, 256, (size_t)9 * k * 4, h->st>>>(labB, nB, k, o.boff, o.perm, o.pos);
  CKL();
  gather_rows_kernel<<<(unsigned)ceil_div(rows, 8), 256, 0, h->st>>>(h->Xhi, h->Xlo, h->norms, h->rscale, o.perm, b0,
                                                                     nB, rows, P.dp, o.hi, o.lo, o.norms, o.rscale);
  CKL();
  return KKM_OK;
}

// The streaming kernel's A operand: rows [row0, row0 + nA) of a split operand with arows rows.
struct StreamA {
  const uint16_t *hi, *lo;
  const float *norms, *rscale;
  int64_t arows, row0, nA, rows_pad;
};

// One fused a1+a2 pass: S[rows_pad][k] (fp64) = the sums over the sorted set B (nB points, brows
// rows, k segments) of kappa(a_i, b_p) by cluster -- accumulated by tc3_stream_kernel in int64 fixed
// point (Sx, exact integer sums in any order, any k in one launch) and converted once. pos (NULL if
// A and B are disjoint): sorted position of A row i for b0 <= i < b0 + npos (the Gaussian
// diagonal). fx = 2^s with nB max|K| 2^s < 2^61.
int stream_pass(kkm_ctx *h, TcStream &ts, const StreamA &A, const SortedSet &B, int64_t brows, int64_t nB,
                int64_t b0, const int32_t *pos, int64_t npos, int splits, double fx, long long *Sx, double *S) {
  const Plan &P = h->P;
  const int k = P.k;
  if (A.nA == 0) return KKM_OK;
  CK(cudaMemsetAsync(Sx, 0, (size_t)A.rows_pad * k * 8, h->st));
  if (tc3_stream_launch(ts, A.hi, A.lo, B.hi, B.lo, P.fp16, A.arows, brows, P.dp, nB, b0, A.row0, A.nA, A.norms,
                        A.rscale, B.norms, B.rscale, pos, npos, B.seg, k, h->kp, splits, fx, Sx, h->st, &h->launches,
                        h->chain_kb)) {
    h->poisoned = true;
    return fail(KKM_ECUDA, "streaming kernel launch failed: %s", tc_gemm_error());
  }
  fx_to_double_kernel<<<(unsigned)ceil_div(A.rows_pad * k, 256), 256, 0, h->st>>>(Sx, A.rows_pad * k, 1.0 / fx, S);
  CKL();
  return KKM_OK;
}

// Streaming a1+a2 of the clustering loop: sort the B set by label, then the fused kernel writes
// the S partials (Spart) of the A set's rows.
int launch_stream(kkm_ctx *h, const int32_t *labels) {
  const Plan &P = h->P;
  const SortedSet B{h->Shi, h->Slo, h->snorms, h->srscale, h->perm, h->pos, h->seg, h->bcount, h->boff};
  CKR(sort_gather(h, labels + P.b0, P.b0, P.nB, P.npad, B));
  const StreamA A{h->Xhi, h->Xlo, h->norms, h->rscale, P.npad, P.a0, P.nA, P.nApad};
  a2_mark(h);
  const int rc = stream_pass(h, h->ts, A, B, P.npad, P.nB, P.b0, h->pos, P.nB, P.stream_splits, h->fx_scale,
                            (long long *)(h->ws + P.o_Sx), h->Spart);
  a2_mark(h);
  return rc;
}

// a2 on the materialised K tile (A set rows x B set columns).
int launch_spmm_mat_body(kkm_ctx *h, const int32_t *labels);
int launch_spmm_mat(kkm_ctx *h, const int32_t *labels) {
  a2_mark(h);
  const int rc = launch_spmm_mat_body(h, labels);
  a2_mark(h);
  return rc;
}

int launch_spmm_mat_body(kkm_ctx *h, const int32_t *labels) {
  const Plan &P = h->P;
  if (P.nA == 0) return KKM_OK;
  if (P.spmm_v2) {
    const int64_t ngroups = P.ldk / 32;
    group_code_kernel<<<(unsigned)ceil_div(ngroups, 8), 256, 0, h->st>>>(labels + P.b0, P.nB, P.ldk, h->codes);
    CKL();
    CK(ensure_smem_attr((const void *)spmm_group_kernel, sg_smem_bytes(SG_MAX_K)));
    const int64_t items = ceil_div(P.nA, SG_ROWS) * P.nsplit;
    const int grid = (int)std::min<int64_t>(items, h->num_sms);
    spmm_group_kernel<<<grid, SG_THREADS, sg_smem_bytes(P.k), h->st>>>(h->K, P.ldk, P.nA, h->codes, P.k, P.nsplit,
                                                                     P.chunks_per_split, P.nApad, h->Spart);
    CKL();
    return KKM_OK;
  }
  if (P.pr > 1) {  // the B set's labels, -1 padded to the tile pitch
    copy_labels_kernel<<<(unsigned)ceil_div(P.ldk, 256), 256, 0, h->st>>>(labels + P.b0, P.nB, P.ldk, h->labB);
    CKL();
    labels = h->labB;
  }
  if (P.k > SP_KPMAX) {
    for (int c0 = 0; c0 < P.k; c0 += SP_KPMAX) CKR(launch_spmm_kp<SP_KPMAX>(h, labels, c0));
    return KKM_OK;
  }
  const int kp = (P.k + 1) / 2 * 2;
  switch (kp) {
    case 2: return launch_spmm_kp<2>(h, labels, 0);
    case 4: return launch_spmm_kp<4>(h, labels, 0);
    case 6: return launch_spmm_kp<6>(h, labels, 0);
    case 8: return launch_spmm_kp<8>(h, labels, 0);
    case 10: return launch_spmm_kp<10>(h, labels, 0);
    case 12: return launch_spmm_kp<12>(h, labels, 0);
    case 14: return launch_spmm_kp<14>(h, labels, 0);
    default: return launch_spmm_kp<16>(h, labels, 0);
  }
}

template <int KP>
int launch_spmm_sym_kp(kkm_ctx *h, const int32_t *labels) {
  const Plan &P = h->P;
  CK(ensure_smem_attr((const void *)spmm_sym_kernel<KP>, spmm_sym_smem_bytes()));
  if (P.sym_items == 0) {
    a2_mark(h);
    a2_mark(h);
    return KKM_OK;
  }
  const int grid = (int)std::min<int64_t>(P.sym_items, h->num_sms);
  a2_mark(h);
  spmm_sym_kernel<KP><<<grid, SYM_THREADS, spmm_sym_smem_bytes(), h->st>>>(
      h->K, h->bands, (int)P.bands.size(), P.sym_items, labels, h->perm_b, h->groups, P.sym_gmax, P.k, P.nApad,
      h->Spart, h->colpart, h->work);
  a2_mark(h);
  CKL();
  return KKM_OK;
}

// f1: a2 over the symmetric band storage -> the rank's contributions to S of all rows (Sfin),
// reduce-scattered over the ranks for P > 1 (each rank then holds S of its own 1D block).
int launch_spmm_sym(kkm_ctx *h, const int32_t *labels, const double **s_out) {
  const Plan &P = h->P;
  const int k = P.k;
  if (P.kh) {  // f4: 16-bit bands, a2 on the tensor cores (spmm_tc.cuh), S in int64 fixed point
    CK(ensure_smem_attr((const void *)spmm_tc_kernel, TS_SMEM));
    long long *Sx = h->tSfix;
    if (h->p2p) {  // this epoch's half of the own exchange buffer (the other half may still be read)
      ++h->epoch;
      Sx = (long long *)(h->xbuf + (h->epoch & 1) * (size_t)P.npad * k * 8);
    }
    CK(cudaMemsetAsync(Sx, 0, (size_t)P.npad * k * 8, h->st));
    a2_mark(h);
    if (!P.tunits.empty()) {
      const int grid = (int)std::min<int64_t>((int64_t)P.tunits.size(), h->num_sms);
      spmm_tc_kernel<<<grid, TS_THREADS, TS_SMEM, h->st>>>(h->tmaps, h->tbands, h->tunits, (int)P.tunits.size(),
                                                           labels, P.n, k, P.npad, h->tfxm, Sx, h->work,
                                                           P.kplanes);
      CKL();
    }
    a2_mark(h);
    if (h->p2p) {  // publish; run_cnorm's finalize sums the ranks' S over NVLink
      peer_signal_kernel<<<1, 1, 0, h->st>>>(
          (unsigned long long *)(h->xbuf + 2 * (size_t)P.npad * k * 8), h->epoch);
      CKL();
      *s_out = nullptr;
      return KKM_OK;
    }
    const unsigned gr = (unsigned)ceil_div(P.npad * k, 256);
    if (P.repl)  // S of all points on every rank (exact int64 sum)
      CKN(ncclAllReduce(h->tSfix, h->tSfix, (size_t)P.npad * k, ncclInt64, ncclSum, h->comm, h->st));
    if (P.a3fix) {  // run_cnorm's finalize reads tSfix directly
      *s_out = nullptr;
      return KKM_OK;
    }
    if (P.nranks == 1 || P.repl) {
      ts_fix_out_kernel<<<gr, 256, 0, h->st>>>(h->tSfix, P.n, P.npad, k, h->tfx_inv, nullptr, h->Sfin);
      CKL();
      *s_out = h->Sfin;
      return KKM_OK;
    }
    // exact: the int64 sums of the ranks' contributions, any order gives the same bits
    ts_fix_out_kernel<<<gr, 256, 0, h->st>>>(h->tSfix, P.n, P.npad, k, 1.0, h->tSint, nullptr);
    CKL();
    CKN(ncclReduceScatter(h->tSint, h->tSmine, (size_t)P.B * k, ncclInt64, ncclSum, h->comm, h->st));
    fx_to_double_kernel<<<(unsigned)ceil_div(P.B * k, 256), 256, 0, h->st>>>(h->tSmine, P.B * k, h->tfx_inv,
                                                                           h->Smine);
    *s_out = h->Smine;
    return KKM_OK;
  }
  band_sort_kernel<<<P.T, SYM_TB, (size_t)(32 * k + 2 * (k + 1)) * 4, h->st>>>(
      labels, P.n, k, sym_rows(k), P.sym_gmax, h->perm_b, h->groups, h->ngroups, h->gfirst);
  CKL();
  int rc;
  switch ((k + 1) / 2 * 2) {
    case 2: rc = launch_spmm_sym_kp<2>(h, labels); break;
    case 4: rc = launch_spmm_sym_kp<4>(h, labels); break;
    case 6: rc = launch_spmm_sym_kp<6>(h, labels); break;
    case 8: rc = launch_spmm_sym_kp<8>(h, labels); break;
    case 10: rc = launch_spmm_sym_kp<10>(h, labels); break;
    case 12: rc = launch_spmm_sym_kp<12>(h, labels); break;
    case 14: rc = launch_spmm_sym_kp<14>(h, labels); break;
    default: rc = launch_spmm_sym_kp<16>(h, labels); break;
  }
  CKR(rc);
  int64_t wmax = 0;
  for (const SymBand &b : P.bands) wmax = std::max<int64_t>(wmax, b.ldb - SYM_TB);
  if (wmax > 0 && !P.bands.empty()) {
    sym_colsum_kernel<<<dim3((unsigned)ceil_div(wmax, 4 * 128), (unsigned)P.bands.size(), (unsigned)k), 128, 0,
                        h->st>>>(
        h->colpart, h->bands, h->gfirst, k, h->colsum);
    CKL();
  }
  sym_reduce_kernel<<<dim3((unsigned)ceil_div(P.npad, 256), (unsigned)k), 256, 0, h->st>>>(
      h->Spart, h->colsum, h->bands, h->band_desc, P.n, P.npad, k, h->Sfin);
  CKL();
  if (P.repl) CKN(ncclAllReduce(h->Sfin, h->Sfin, (size_t)P.npad * k, ncclDouble, ncclSum, h->comm, h->st));
  if (P.nranks == 1 || P.repl) {
    *s_out = h->Sfin;
    return KKM_OK;
  }
  CKN(ncclReduceScatter(h->Sfin, h->Smine, (size_t)P.B * k, ncclDouble, ncclSum, h->comm, h->st));
  *s_out = h->Smine;
  return KKM_OK;
}

// f1 streaming a1+a2: sort all points by label, the upper-triangle kernel accumulates S of
// the sorted points in int64 fixed point; back to original order (exact), reduce-scattered
// in int64 for P > 1 (exact: any reduction order gives the same bits), then fp64.
int launch_stream_sym(kkm_ctx *h, const int32_t *labels, const double **s_out) {
  const Plan &P = h->P;
  const int k = P.k;
  const SortedSet B{h->Shi, h->Slo, h->snorms, h->srscale, h->perm, h->pos, h->seg, h->bcount, h->boff};
  CKR(sort_gather(h, labels, 0, P.n, P.npad, B));
  CK(cudaMemsetAsync(h->Sfix, 0, (size_t)P.npad * k * 8, h->st));
  a2_mark(h);
  int rc = ssym_launch(h->ts, h->Shi, h->Slo, P.fp16, P.npad, P.dp, P.n, h->snorms, h->srscale, h->seg, k, h->kp,
                       h->units, (int64_t)P.units.size(), h->fx_scale, h->Sfix, h->st, &h->launches, h->chain_kb);
  a2_mark(h);
  if (rc) {
    h->poisoned = true;
    return fail(KKM_ECUDA, "symmetric streaming kernel launch failed: %s", tc_gemm_error());
  }
  const unsigned g = (unsigned)ceil_div(P.npad * k, 256);
  double *Sd = h->Spart;  // P.nsplit = 1: [npad][k] fp64
  if (P.repl)  // the sorted order is the same on every rank (same labels, stable sort): sum in place
    CKN(ncclAllReduce(h->Sfix, h->Sfix, (size_t)P.npad * k, ncclInt64, ncclSum, h->comm, h->st));
  if (P.nranks == 1 || P.repl) {
    fx_unpermute_kernel<<<g, 256, 0, h->st>>>(h->Sfix, h->pos, P.n, P.npad, k, h->fx_inv, nullptr, Sd);
    CKL();
    *s_out = Sd;
    return KKM_OK;
  }
  fx_unpermute_kernel<<<g, 256, 0, h->st>>>(h->Sfix, h->pos, P.n, P.npad, k, h->fx_inv, h->Sorig, nullptr);
  CKL();
  CKN(ncclReduceScatter(h->Sorig, h->Sfmine, (size_t)P.B * k, ncclInt64, ncclSum, h->comm, h->st));
  fx_to_double_kernel<<<(unsigned)ceil_div(P.B * k, 256), 256, 0, h->st>>>(h->Sfmine, P.B * k, h->fx_inv, h->Smine);
  CKL();
  *s_out = h->Smine;
  return KKM_OK;
}

// a2 + the 1.5D column-split reduce-scatter: afterwards the S partials of this rank's own 1D
// block are in s_out[nsplit_out][B][k] (the 1D case reduces nothing: s_out = Spart).
int launch_spmm(kkm_ctx *h, const int32_t *labels, const double **s_out, int *nsplit_out) {
  const Plan &P = h->P;
  if (P.sym) {
    *nsplit_out = 1;
    return launch_spmm_sym(h, labels, s_out);
  }
  if (P.ssym) {
    *nsplit_out = 1;
    return launch_stream_sym(h, labels, s_out);
  }
  CKR(P.materialize ? launch_spmm_mat(h, labels) : launch_stream(h, labels));
  if (P.pr == 1) {
    *s_out = h->Spart;
    *nsplit_out = P.nsplit;
    return KKM_OK;
  }
  split_sum_kernel<<<(unsigned)ceil_div(P.nApad * P.k, 256), 256, 0, h->st>>>(h->Spart, P.nsplit, P.nA,
                                                                              P.nApad, P.k, h->Scol);
  CKL();
  // P(i, j) keeps piece i of column block j = its own 1D block (column-major ranks)
  CKN(ncclReduceScatter(h->Scol, h->Smine, (size_t)P.B * P.k, ncclDouble, ncclSum, h->colcomm, h->st));
  *s_out = h->Smine;
  *nsplit_out = 1;
  return KKM_OK;
}

// a3: E, z, c (cnorm) and J for the labels entering the iteration -> E_out, cnorm_out,
// J_out. sizes_next / changed_out (may be NULL) are zeroed for the following assign.
int run_cnorm(kkm_ctx *h, const double *S, int nsplit, int64_t rows_pad, double *E_out, double *cnorm_out,
              double *J_out, int32_t *sizes_next, unsigned long long *changed_out) {
  const Plan &P = h->P;
  const int32_t *labels = h->lab[h->cur];
  const int32_t *sizes = h->sizes[h->cur];
  const int k1 = P.k + 1;
  const int nr = P.repl ? 1 : P.nranks, r = P.repl ? 0 : P.rank;  // replicated a3: one "rank"
  if (P.a3fix && P.a_n > 0) {  // int64 S in, c and J from the last block (same sums as below)
    const int fth = fin_threads(P.k);
    const A3Peers peers = h->p2p ? A3Peers{h->xtable, P.nranks, (int64_t)((h->epoch & 1) * (size_t)P.npad * P.k * 8),
                                           (int64_t)h->xflag_off, h->epoch, h->p2p_timeout_ns,
                                           (int *)(h->xbuf + h->xflag_off + 64)}
                                 : A3Peers{nullptr, 0, 0, 0, 0ull, 0ull, nullptr};
    finalize_kernel<<<P.nfin, fth, (size_t)k1 * fth * 8, h->st>>>(
        nullptr, 1, P.a_n, P.npad, P.k, sizes, labels + P.a_row0, h->diag, P.rows_per_block, E_out, h->blockpart,
        h->tSfix, h->tfx_inv, A3Fused{h->a3ctr, sizes, cnorm_out, J_out, sizes_next, changed_out}, peers);
    CKL();
    return KKM_OK;
  }
  if (P.a_n > 0) {
    const int fth = fin_threads(P.k);
    finalize_kernel<<<P.nfin, fth, (size_t)k1 * fth * 8, h->st>>>(
        S, nsplit, P.a_n, rows_pad, P.k, sizes, labels + P.a_row0, h->diag, P.rows_per_block,
        E_out, h->blockpart);
    CKL();
  }
  cnorm_local_kernel<<<1, 32 * std::min(32, k1), 0, h->st>>>(h->blockpart, P.a_n > 0 ? P.nfin : 0, P.k,
                                           h->rankpart + (int64_t)r * k1);
  CKL();
  if (nr > 1)
    CKN(ncclAllGather(h->rankpart + (int64_t)r * k1, h->rankpart, k1, ncclDouble, h->comm, h->st));
  cnorm_final_kernel<<<1, 128, 0, h->st>>>(h->rankpart, nr, P.k, sizes, cnorm_out, J_out,
                                           sizes_next, changed_out);
  CKL();
  return KKM_OK;
}

// a4 + the V update: new labels into lab[cur^1], sizes into sizes[cur^1], allgather.
int run_assign(kkm_ctx *h, unsigned long long *changed_out) {
  const Plan &P = h->P;
  const int nx = h->cur ^ 1;
  if (P.a_n > 0) {
    const int th = 256;
    assign_kernel<<<(unsigned)ceil_div(P.a_n, th), th, (size_t)P.k * 4, h->st>>>(
        h->E, P.a_n, P.k, h->cnorm, h->diag, h->lab[h->cur] + P.a_row0, h->lab[nx] + P.a_row0,
        h->sizes[nx], changed_out, h->Dfull);
    CKL();
  }
  if (P.nranks > 1 && !P.repl) {  // the changed count is global too: every rank takes the same control path
    CKN(ncclGroupStart());
    CKN(ncclAllGather(h->lab[nx] + P.row0, h->lab[nx], P.B, ncclInt32, h->comm, h->st));
    CKN(ncclAllReduce(h->sizes[nx], h->sizes[nx], P.k, ncclInt32, ncclSum, h->comm, h->st));
    CKN(ncclAllReduce(changed_out, changed_out, 1, ncclUint64, ncclSum, h->comm, h->st));
    CKN(ncclGroupEnd());
  }
  return KKM_OK;
}

// oscale > 0: out is fp16 and receives K * oscale (tensor-core precisions only)
int launch_gemm(kkm_ctx *h, int64_t i0, int64_t m, int64_t j0, int64_t ncov, void *out, int64_t ldo,
                float oscale = 0.f, void *out_lo = nullptr) {
  const Plan &P = h->P;
  if (m <= 0 || ncov <= 0) return KKM_OK;
  if (P.tc) {
    int rc = tc3_gemm_launch(h->tc, h->Xhi, h->Xlo, P.fp16, h->rscale, P.npad, P.dp, P.n, i0, m, j0, ncov, h->norms,
                             h->kp, out, ldo, h->st, &h->launches, oscale, out_lo, h->chain_kb);
    if (rc) {
      h->poisoned = true;
      return fail(KKM_ECUDA, "tcgen05 GEMM launch failed: %s", tc_gemm_error());
    }
    return KKM_OK;
  }
  dim3 grid((unsigned)ceil_div(ncov, SG_BN), (unsigned)ceil_div(m, SG_BM));
  gemm_simt_kernel<<<grid, 256, 0, h->st>>>(h->Xf, P.ldf, P.n, P.d, i0, m, j0, ncov, h->norms,
                                             h->kp, (float *)out, ldo);
  CKL();
  return KKM_OK;
}

// f3: S of the own rows for the labels lab[cur ^ 1] from S (Sinc) of lab[cur]: the points
// that moved, sorted by new label, added; sorted by old label, subtracted (the fused
// streaming kernel, A = own rows, B = the moved points). m = number of moved points.
int delta_update(kkm_ctx *h, int64_t m) {
  const Plan &P = h->P;
  const int k = P.k;
  const int32_t *cl_old = h->lab[h->cur], *cl_new = h->lab[h->cur ^ 1];
  const int nblk = (int)ceil_div(P.n, SORT_BLOCK);
  const int64_t mpad = round_up(m, 256);
  const int splits = std::min(8, ts_choose_splits((P.nloc + 1) / 2, m, h->num_sms / 2));
  const StreamA A{h->Xhi, h->Xlo, h->norms, h->rscale, P.npad, P.row0, P.nloc, P.B};
  for (int pass = 0; pass < 2; ++pass) {  // 0: + new labels, 1: - old labels
    moved_key_kernel<<<(unsigned)ceil_div(P.lablen, 256), 256, 0, h->st>>>(cl_old, cl_new, P.n, P.lablen, k,
                                                                           pass == 0, h->dkey);
    CKL();
    const SortedSet &D = h->dset;
    sort_count_kernel<<<nblk, 256, (size_t)(k + 1) * 4, h->st>>>(h->dkey, P.n, k + 1, D.bcount);
    CKL();
    sort_scan_kernel<<<k + 2, 1024, 1024 * 4, h->st>>>(D.bcount, nblk, k + 1, D.boff, D.seg);
    CKL();
    sort_scatter_kernel<<<nblk, 256, (size_t)9 * (k + 1) * 4, h->st>>>(h->dkey, P.n, k + 1, D.boff, D.perm, D.pos);
    CKL();
    gather_rows_kernel<<<(unsigned)ceil_div(mpad, 8), 256, 0, h->st>>>(h->Xhi, h->Xlo, h->norms, h->rscale, D.perm, 0,
                                                                       m, mpad, P.dp, D.hi, D.lo, D.norms, D.rscale);
    CKL();
    // B = the m moved points (clusters 0..k-1 of the k+1 buckets); pos: sorted position of
    // each point (>= m for the points that did not move) for the Gaussian diagonal
    CKR(stream_pass(h, h->ts_delta, A, D, mpad, m, 0, D.pos, P.n, splits, h->fx_scale, h->Sdx, h->Sd));
    sinc_add_kernel<<<(unsigned)ceil_div(P.nloc * k, 256), 256, 0, h->st>>>(h->Sd, 1, P.B, P.nloc, k,
                                                                            pass == 0 ? 1.0 : -1.0, h->Sinc);
    CKL();
  }
  return KKM_OK;
}

struct EvPair {
  cudaEvent_t a = nullptr, b = nullptr;
};

}  // namespace

extern "C" {

int kkm_default_params(kkm_params *p) {
  if (!p) return fail(KKM_EINVAL, "params is NULL");
  std::memset(p, 0, sizeof(*p));
  p->kind = KKM_KERNEL_POLY;
  p->gamma = 1.0;
  p->coef0 = 1.0;
  p->degree = 2;
  p->k = 2;
  p->max_iter = 100;
  p->path = KKM_PATH_AUTO;
  p->precision = KKM_PREC_FP16X3;
  return KKM_OK;
}

int64_t kkm_shard_begin(int64_t n, int32_t rank, int32_t nranks) {
  if (nranks < 1 || n < 0 || rank < 0) return -1;
  const int64_t B = ceil_div(n, nranks);
  return std::min<int64_t>(n, (int64_t)rank * B);
}

int kkm_workspace_size(const kkm_params *p, int64_t n, int64_t d, int32_t rank, int32_t nranks,
                       size_t *bytes) {
  if (!bytes) return fail(KKM_EINVAL, "bytes is NULL");
  Plan P;
  CKR(make_plan(p, n, d, rank, nranks, &P));
  *bytes = P.total;
  return KKM_OK;
}

int kkm_plan_query(const kkm_params *p, int64_t n, int64_t d, int32_t rank, int32_t nranks, kkm_plan_info *info,
                   int64_t *pieces, int64_t cap) {
  if (!info) return fail(KKM_EINVAL, "info is NULL");
  Plan P;
  CKR(make_plan(p, n, d, rank, nranks, &P));
  std::memset(info, 0, sizeof(*info));
  info->path = P.materialize ? KKM_PATH_MATERIALIZE : KKM_PATH_STREAM;
  info->layout = P.sym ? (P.kh ? KKM_LAYOUT_SYM_BANDS16 : KKM_LAYOUT_SYM_BANDS)
                 : P.ssym ? KKM_LAYOUT_SYM_STREAM : P.materialize ? KKM_LAYOUT_FULL : KKM_LAYOUT_STREAM;
  info->exchange = nranks == 1 ? KKM_XCHG_NONE
                   : P.repl ? KKM_XCHG_S_ALLREDUCE
                   : (P.sym || P.ssym) ? KKM_XCHG_S_REDUCE_SCATTER : KKM_XCHG_PARTIALS;
  info->grid_rows = P.pr;
  info->grid_cols = P.pc;
  info->row0 = P.row0;
  info->nloc = P.nloc;
  info->a0 = P.a0;
  info->nA = P.nA;
  info->b0 = P.b0;
  info->nB = P.nB;
  info->ws_bytes = (int64_t)P.total;
  std::vector<int64_t> r;
  auto add = [&](int64_t r0, int64_t nr, int64_t c0, int64_t nc, int64_t cd) {
    nr = std::min(nr, n - r0);
    nc = std::min(nc, n - c0);
    if (nr <= 0 || nc <= 0) return;
    r.insert(r.end(), {r0, nr, c0, nc, std::min(cd, n)});
  };
  if (P.sym) {
    for (const SymBand &b : P.bands) {
      const int64_t j0 = (int64_t)b.band * SYM_TB;
      add(j0 + b.row0, b.rows, j0, n - j0, j0 + SYM_TB);
    }
  } else if (P.ssym) {
    for (const int4 &u : P.units) add((int64_t)u.x * 256, 256, (int64_t)u.y * 256, (int64_t)u.z * 256,
                                      u.x == u.y ? (int64_t)(u.y + 1) * 256 : (int64_t)u.y * 256);
  } else {
    add(P.a0, P.nA, P.b0, P.nB, n);
  }
  info->npieces = (int64_t)(r.size() / 5);
  if (pieces)
    std::memcpy(pieces, r.data(), (size_t)std::min<int64_t>(cap, info->npieces) * 5 * sizeof(int64_t));
  return KKM_OK;
}

const char *kkm_last_error(void) { return g_err; }

// *v = the minimum of *v over all ranks (a collective on the handle's communicator).
static int agree_min(kkm_ctx *h, int *v) {
  int *d = nullptr;
  if (cudaMallocAsync((void **)&d, 4, h->st) != cudaSuccess) return fail(KKM_ECUDA, "cudaMallocAsync failed");
  int rc = [&]() -> int {
    CK(cudaMemcpyAsync(d, v, 4, cudaMemcpyHostToDevice, h->st));
    CKN(ncclAllReduce(d, d, 1, ncclInt32, ncclMin, h->comm, h->st));
    CK(cudaMemcpyAsync(v, d, 4, cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    return KKM_OK;
  }();
  cudaFreeAsync(d, h->st);
  return rc;
}

// After a synchronised a3 on the peer path: a finalize that gave up waiting for a peer poisons the
// handle (KKM_ENCCL: the exchange failed) instead of trapping the context.
static int check_p2p(kkm_ctx *h) {
  if (!h->p2p) return KKM_OK;
  int to = 0;
  CK(cudaMemcpy(&to, h->xbuf + h->xflag_off + 64, 4, cudaMemcpyDeviceToHost));
  if (to) {
    h->poisoned = true;
    return fail(KKM_ENCCL, "peer-memory S exchange: a peer's flag did not arrive within %.0f s",
                (double)h->p2p_timeout_ns * 1e-9);
  }
  return KKM_OK;
}

// Peer-memory exchange of S for the replicated a3 (16-bit bands, several ranks, §6): an own
// cudaMalloc'd buffer [2 epochs of k x npad int64 | epoch flag | peer table], its IPC handle
// allgathered over NCCL and the peers' buffers opened here. All ranks must agree: the outcome is
// allreduced (min) and any failure leaves every rank on the NCCL allreduce path. Collective.
static int setup_p2p(kkm_ctx *h) {
  const Plan &P = h->P;
  const size_t sbytes = (size_t)P.npad * P.k * 8;
  const size_t xbytes = 2 * sbytes + 256 + (size_t)P.nranks * 8;
  int ok = 1;
  char *dh = nullptr;
  std::vector<char> hs((size_t)64 * P.nranks);
  std::vector<const uint8_t *> bases((size_t)P.nranks, nullptr);
  if (cudaMalloc(&h->xbuf, xbytes) != cudaSuccess) {
    h->xbuf = nullptr;
    ok = 0;
  }
  if (ok && cudaMemset(h->xbuf, 0, xbytes) != cudaSuccess) ok = 0;
  cudaIpcMemHandle_t mine;
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  if (ok && cudaIpcGetMemHandle(&mine, h->xbuf) != cudaSuccess) ok = 0;
  if (cudaMalloc(&dh, hs.size() + 8) != cudaSuccess) return fail(KKM_ECUDA, "cudaMalloc (IPC handles) failed");
  if (ok) CK(cudaMemcpy(dh + 64 * (size_t)P.rank, &mine, 64, cudaMemcpyHostToDevice));
  CKN(ncclAllGather(dh + 64 * (size_t)P.rank, dh, 64, ncclChar, h->comm, h->st));
  CK(cudaMemcpyAsync(hs.data(), dh, hs.size(), cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  if (ok) {
    for (int r = 0; r < P.nranks; ++r) {
      if (r == P.rank) {
        bases[(size_t)r] = h->xbuf;
        continue;
      }
      cudaIpcMemHandle_t hr;
      std::memcpy(&hr, hs.data() + 64 * (size_t)r, 64);
      void *q = nullptr;
      if (cudaIpcOpenMemHandle(&q, hr, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
        cudaGetLastError();
        ok = 0;
        break;
      }
      h->xpeers.push_back(q);
      bases[(size_t)r] = (const uint8_t *)q;
    }
  }
  // every rank on the same path
  int *dok = (int *)(dh + hs.size());
  CK(cudaMemcpy(dok, &ok, 4, cudaMemcpyHostToDevice));
  CKN(ncclAllReduce(dok, dok, 1, ncclInt32, ncclMin, h->comm, h->st));
  CK(cudaMemcpyAsync(&ok, dok, 4, cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  cudaFree(dh);
  if (ok) {
    h->xtable = (const uint8_t **)(h->xbuf + 2 * sbytes + 256);
    h->xflag_off = 2 * sbytes;
    CK(cudaMemcpy((void *)h->xtable, bases.data(), (size_t)P.nranks * 8, cudaMemcpyHostToDevice));
    h->p2p = true;
    return KKM_OK;
  }
  for (void *q : h->xpeers) cudaIpcCloseMemHandle(q);
  h->xpeers.clear();
  if (h->xbuf) cudaFree(h->xbuf);
  h->xbuf = nullptr;
  cudaGetLastError();
  return KKM_OK;  // NCCL allreduce path
}

int kkm_init(kkm_handle *out, const kkm_params *p, const float *X_local, int64_t n, int64_t d,
             int64_t ldx, int32_t rank, int32_t nranks, const int32_t *init_labels, void *workspace,
             size_t ws_bytes, void *cuda_stream, void *nccl_comm) {
  if (!out) return fail(KKM_EINVAL, "out is NULL");
  *out = nullptr;
  Plan P;
  CKR(make_plan(p, n, d, rank, nranks, &P));
  if (ldx < d) return fail(KKM_EINVAL, "ldx=%lld < d=%lld", (long long)ldx, (long long)d);
  if (!X_local && P.nloc > 0) return fail(KKM_EINVAL, "X_local is NULL");
  if (!workspace) return fail(KKM_EINVAL, "workspace is NULL");
  if (((uintptr_t)workspace) & 255) return fail(KKM_EINVAL, "workspace must be 256-byte aligned");
  if (ws_bytes < P.total)
    return fail(KKM_ENOMEM, "workspace %zu bytes < required %zu", ws_bytes, P.total);
  if (nranks > 1 && !nccl_comm) return fail(KKM_EINVAL, "nranks > 1 needs an NCCL communicator");

  kkm_ctx *h = new kkm_ctx();
  h->p = *p;
  h->P = P;
  h->st = (cudaStream_t)cuda_stream;
  h->comm = (ncclComm_t)nccl_comm;
  h->ws = (uint8_t *)workspace;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
    delete h;
    return fail(KKM_ECUDA, "no CUDA device");
  }
  uint8_t *w = h->ws;
  h->Xf = (float *)(w + P.o_Xf);
  h->mean = (float *)(w + P.o_mean);
  h->Xhi = P.tc ? (uint16_t *)(w + P.o_Xhi) : nullptr;
  h->Xlo = P.tc ? (uint16_t *)(w + P.o_Xlo) : nullptr;
  h->rscale = (float *)(w + P.o_rscale);
  h->norms = (float *)(w + P.o_norms);
  h->diag = (double *)(w + P.o_diag);
  h->K = P.materialize ? (float *)(w + P.o_K) : nullptr;
  for (int b = 0; b < 2; ++b) {
    h->lab[b] = (int32_t *)(w + P.o_lab[b]);
    h->sizes[b] = (int32_t *)(w + P.o_sizes[b]);
  }
  h->Spart = (double *)(w + P.o_Spart);
  h->E = (double *)(w + P.o_E);
  h->a3ctr = (unsigned *)(w + P.o_a3ctr);
  h->blockpart = (double *)(w + P.o_blockpart);
  h->rankpart = (double *)(w + P.o_rankpart);
  h->cnorm = (double *)(w + P.o_cnorm);
  h->J = (double *)(w + P.o_J);
  h->changed = (unsigned long long *)(w + P.o_changed);
  h->Dfull = (double *)(w + P.o_Dfull);
  h->bad = (int *)(w + P.o_bad);
  h->E2 = (double *)(w + P.o_E2);
  h->cnorm2 = (double *)(w + P.o_cnorm2);
  if (!P.materialize) {
    h->Shi = (uint16_t *)(w + P.o_Shi);
    h->Slo = (uint16_t *)(w + P.o_Slo);
    h->snorms = (float *)(w + P.o_snorms);
    h->srscale = (float *)(w + P.o_srscale);
    h->perm = (int32_t *)(w + P.o_perm);
    h->pos = (int32_t *)(w + P.o_pos);
    h->seg = (int32_t *)(w + P.o_seg);
    h->bcount = (int32_t *)(w + P.o_bcount);
    h->boff = (int32_t *)(w + P.o_boff);
  }
  h->fxmax = (float *)(w + P.o_fxmax);
  if (P.materialize && P.spmm_v2) h->codes = (uint32_t *)(w + P.o_codes);
  if (P.pr > 1) {
    h->labB = (int32_t *)(w + P.o_labB);
    h->Scol = (double *)(w + P.o_Scol);
  }
  if (P.need_smine) h->Smine = (double *)(w + P.o_Smine);
  if (P.inc) {
    h->Sinc = (double *)(w + P.o_Sinc);
    h->Sd = (double *)(w + P.o_Sd);
    h->Sdx = (long long *)(w + P.o_Sdx);
    h->dkey = (int32_t *)(w + P.o_dkey);
    h->dset = SortedSet{(uint16_t *)(w + P.o_Dhi), (uint16_t *)(w + P.o_Dlo), (float *)(w + P.o_Dn),
                        (float *)(w + P.o_Dr),      (int32_t *)(w + P.o_dperm), (int32_t *)(w + P.o_dpos),
                        (int32_t *)(w + P.o_dseg),  (int32_t *)(w + P.o_dbc),   (int32_t *)(w + P.o_dbo)};
  }
  if (P.ssym) {
    h->units = (int4 *)(w + P.o_units);
    h->Sfix = (long long *)(w + P.o_Sfix);
    if (P.nranks > 1) {
      h->Sorig = (long long *)(w + P.o_Sorig);
      h->Sfmine = (long long *)(w + P.o_Sfmine);
    }
  }
  if (P.sym) {
    h->perm_b = (int32_t *)(w + P.o_perm_b);
    h->groups = (SymGroup *)(w + P.o_groups);
    h->ngroups = (int32_t *)(w + P.o_ngroups);
    h->bands = (SymBand *)(w + P.o_bands);
    h->band_desc = (int32_t *)(w + P.o_band_desc);
    h->colpart = (float *)(w + P.o_colpart);
    h->colsum = (double *)(w + P.o_colsum);
    h->work = (int32_t *)(w + P.o_work);
    if (P.kh) {
      h->tmaps = (CUtensorMap *)(w + P.o_tmaps);
      h->tbands = (TsBand *)(w + P.o_tbands);
      h->tunits = (TsUnit *)(w + P.o_tunits);
      h->tSfix = (long long *)(w + P.o_tSfix);
      if (P.nranks > 1) {
        h->tSint = (long long *)(w + P.o_tSint);
        h->tSmine = (long long *)(w + P.o_tSmine);
      }
    }
    h->gfirst = (int32_t *)(w + P.o_gfirst);
    h->Sfin = (double *)(w + P.o_Sfin);
  }
  if (const char *e = std::getenv("KKM_CHAIN_KB")) h->chain_kb = std::max(0, std::atoi(e));
  h->kp.kind = p->kind;
  h->kp.degree = p->degree;
  h->kp.gamma = (float)p->gamma;
  h->kp.coef0 = (float)p->coef0;
  h->kp.neg_gamma_log2e = (float)(-p->gamma * 1.4426950408889634);

  int rc = [&]() -> int {
    if (P.fused) CK(ensure_smem_attr((const void *)fused_update_kernel, 17 * FUSED_THREADS * 8 + 16 * 8));
    if (fin_smem_bytes(P.k) > 48 * 1024) CK(ensure_smem_attr((const void *)finalize_kernel, fin_smem_bytes(P.k)));
    EventList evs;  // init phases: prep, GEMM
    if (!evs.record(h->st)) return fail(KKM_ECUDA, "cudaEventCreate/Record failed");
    // ---- X (Alg. 1 line 1: allgather P) into Xf [npad x ldf], zero padded
    CK(cudaMemsetAsync(h->Xf, 0, (size_t)P.npad * P.ldf * 4, h->st));
    if (P.nloc > 0)
      CK(cudaMemcpy2DAsync(h->Xf + P.row0 * P.ldf, P.ldf * 4, X_local, ldx * 4, P.d * 4, P.nloc,
                           cudaMemcpyDefault, h->st));
    if (P.nranks > 1)
      CKN(ncclAllGather(h->Xf + (int64_t)P.rank * P.B * P.ldf, h->Xf, (size_t)P.B * P.ldf, ncclFloat,
                        h->comm, h->st));
    // ---- Gaussian: center X on its column means (exact for kappa; smaller norms shrink the
    // accumulation bias of r^2 on the tensor cores, DESIGN A9). Every rank holds all of X.
    CK(cudaMemsetAsync(h->mean, 0, (size_t)P.ldf * 4, h->st));
    if (p->kind == KKM_KERNEL_GAUSSIAN) {
      const unsigned nch = (unsigned)ceil_div(P.n, CM_ROWS);
      double *part = (double *)(h->ws + P.o_cmpart);
      colmean_partial_kernel<<<dim3((unsigned)ceil_div(P.d, 128), nch), 128, 0, h->st>>>(h->Xf, P.ldf, P.n, P.d, part);
      CKL();
      colmean_final_kernel<<<(unsigned)ceil_div(P.d, 128), 128, 0, h->st>>>(part, (int)nch, P.n, P.d, h->mean);
      CKL();
      center_rows_kernel<<<(unsigned)ceil_div(P.n, 8), 256, 0, h->st>>>(h->Xf, P.ldf, P.n, P.d, h->mean);
      CKL();
    }
    // ---- a5: norms, bf16 split, diag
    {
      const int wpb = 8;
      prep_rows_kernel<<<(unsigned)ceil_div(P.npad, wpb), wpb * 32, 0, h->st>>>(
          h->Xf, P.ldf, P.n, P.npad, P.d, h->norms, h->Xhi, h->Xlo, P.dp,
          P.tc ? (P.fp16 ? 2 : 1) : 0, h->rscale);
      CKL();
      // Gaussian: the norms of r^2 = n_i + n_j - 2 b become the tensor core's own x_i . x_i, so the
      // one-signed accumulation error of b and of the norms cancels for like terms (DESIGN A9)
      if (p->kind == KKM_KERNEL_GAUSSIAN && P.tc &&
          tc3_self_dots(h->tc, h->Xhi, h->Xlo, P.fp16, h->rscale, P.npad, P.dp, P.n, h->norms, h->st, &h->launches,
                        h->chain_kb)) {
        h->poisoned = true;
        return fail(KKM_ECUDA, "tensor-core self dots failed: %s", tc_gemm_error());
      }
      if (P.a_n > 0) {
        diag_kernel<<<(unsigned)ceil_div(P.a_n, wpb), wpb * 32, 0, h->st>>>(
            h->Xf, P.ldf, P.d, P.a_row0, P.a_n, p->kind, p->gamma, p->coef0, p->degree, h->diag);
        CKL();
      }
    }
    // ---- labels (A5 round robin, or the caller's) and sizes
    for (int b = 0; b < 2; ++b) {
      round_robin_kernel<<<(unsigned)ceil_div(P.lablen, 256), 256, 0, h->st>>>(h->lab[b], P.n, P.lablen, P.k);
      CKL();
    }
    if (init_labels) {
      CK(cudaMemsetAsync(h->bad, 0, 4, h->st));
      int32_t *tmp = h->lab[1];
      CK(cudaMemcpyAsync(tmp, init_labels, (size_t)P.n * 4, cudaMemcpyDefault, h->st));
      load_labels_kernel<<<(unsigned)ceil_div(P.lablen, 256), 256, 0, h->st>>>(tmp, h->lab[0], P.n,
                                                                               P.lablen, P.k, h->bad);
      CKL();
      round_robin_kernel<<<(unsigned)ceil_div(P.lablen, 256), 256, 0, h->st>>>(h->lab[1], P.n, P.lablen, P.k);
      CKL();
      int bad = 0;
      CK(cudaMemcpyAsync(&bad, h->bad, 4, cudaMemcpyDeviceToHost, h->st));
      CK(cudaStreamSynchronize(h->st));
      if (bad) return fail(KKM_ELABEL, "%d init labels outside [0, %d)", bad, P.k);
    }
    CK(cudaMemsetAsync(h->sizes[0], 0, (size_t)P.k * 4, h->st));
    histogram_kernel<<<std::min<int64_t>(ceil_div(P.n, 256), 1024), 256, (size_t)P.k * 4, h->st>>>(
        h->lab[0], P.n, P.k, h->sizes[0]);
    CKL();
    if (!evs.record(h->st)) return fail(KKM_ECUDA, "cudaEventCreate/Record failed");
    // ---- a1: K tile [A set, B set] = kappa(X X^T), materialised once; with
    // symmetric storage (f1) the owned upper-triangle bands, one launch each
    if (P.ssym && !P.units.empty())
      CK(cudaMemcpyAsync(h->units, P.units.data(), P.units.size() * sizeof(int4), cudaMemcpyHostToDevice, h->st));
    if (P.tc) {  // the fixed-point scale 2^s of the streaming kernels' S (loop, f3 deltas): n max|K| 2^s < 2^61
      max_norm_kernel<<<1, 1024, 0, h->st>>>(h->norms, P.n, h->fxmax);
      CKL();
      float mx = 0.f;
      CK(cudaMemcpyAsync(&mx, h->fxmax, 4, cudaMemcpyDeviceToHost, h->st));
      CK(cudaStreamSynchronize(h->st));
      // |K_ij| <= max_i K_ii (K is a Gram matrix of phi); K_ii from the squared norm
      double kmax = 1.0;
      if (p->kind == KKM_KERNEL_LINEAR) kmax = std::max(1e-30, (double)mx);
      if (p->kind == KKM_KERNEL_POLY) kmax = std::pow(p->gamma * mx + std::fabs(p->coef0), (double)p->degree);
      const int sh = (int)std::floor(61.0 - std::log2(std::max(1e-300, (double)P.n * kmax * 1.0001)));
      h->fx_scale = std::ldexp(1.0, sh);
      h->fx_inv = std::ldexp(1.0, -sh);
    }
    if (P.sym) {
      if (!P.bands.empty())
        CK(cudaMemcpyAsync(h->bands, P.bands.data(), P.bands.size() * sizeof(SymBand), cudaMemcpyHostToDevice,
                           h->st));
      CK(cudaMemcpyAsync(h->band_desc, P.band_desc.data(), (size_t)P.T * 4, cudaMemcpyHostToDevice, h->st));
      CK(cudaMemsetAsync(h->work, 0, 2 * 4, h->st));
      CK(cudaMemsetAsync(h->a3ctr, 0, 16, h->st));
      if (P.kh) {  // f4: storage scale 2^e with |K| 2^e <= 60000 (|K_ij| <= max_i K_ii, bounded as for ssym)
        max_norm_kernel<<<1, 1024, 0, h->st>>>(h->norms, P.n, h->fxmax);
        CKL();
        float mx = 0.f;
        CK(cudaMemcpyAsync(&mx, h->fxmax, 4, cudaMemcpyDeviceToHost, h->st));
        CK(cudaStreamSynchronize(h->st));
        double kmax = 1.0;
        if (p->kind == KKM_KERNEL_LINEAR) kmax = (double)mx;
        if (p->kind == KKM_KERNEL_POLY) kmax = std::pow(p->gamma * mx + std::fabs(p->coef0), (double)p->degree);
        const int e = std::max(-100, std::min(100, (int)std::floor(std::log2(60000.0 / std::max(1e-30, kmax * 1.0001)))));
        h->kscale = std::ldexp(1.0f, e);
        // S as int64 fixed point 2^s with n max|K| 2^s < 2^61 (as the streaming f1 kernel)
        const int sh = (int)std::floor(61.0 - std::log2(std::max(1e-300, (double)P.n * kmax * 1.0001)));
        h->tfxm = std::ldexp(1.0, sh - e);
        h->tfx_inv = std::ldexp(1.0, -sh);
        std::vector<CUtensorMap> maps(P.tbands.size() * P.kplanes);
        for (size_t b = 0; b < P.tbands.size(); ++b)
          for (int pl = 0; pl < P.kplanes; ++pl)
            if (ts_encode_band(&maps[b * P.kplanes + pl], (const __half *)h->K + pl * P.kelems + P.tbands[b].koff,
                               P.tbands[b].rows, P.tbands[b].ldb))
              return fail(KKM_ECUDA, "%s", tc_gemm_error());
        if (!maps.empty()) {
          CK(cudaMemcpyAsync(h->tmaps, maps.data(), maps.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice, h->st));
          CK(cudaMemcpyAsync(h->tbands, P.tbands.data(), P.tbands.size() * sizeof(TsBand), cudaMemcpyHostToDevice,
                             h->st));
        }
        if (!P.tunits.empty())
          CK(cudaMemcpyAsync(h->tunits, P.tunits.data(), P.tunits.size() * sizeof(TsUnit), cudaMemcpyHostToDevice,
                             h->st));
        CK(cudaStreamSynchronize(h->st));  // (host vectors go out of scope)
      }
      if (P.tc && !P.bands.empty()) {  // all owned pieces in one tcgen05 launch
        const int planes = P.kh ? P.kplanes : 1;
        std::vector<T2Region> regs(P.bands.size());
        std::vector<CUtensorMap> maps(P.bands.size() * planes);
        int64_t items = 0;
        for (size_t r = 0; r < P.bands.size(); ++r) {
          const SymBand &b = P.bands[r];
          T2Region &g = regs[r];
          g.j0 = (int64_t)b.band * SYM_TB;  // rows of the piece, columns >= the band start
          g.i0 = g.j0 + b.row0;
          g.m = b.rows;
          g.ncov = b.ldb;
          g.item0 = items;
          g.tiles_m = (int32_t)ceil_div(b.rows, T2_BM);
          g.tiles_n = (int32_t)ceil_div(b.ldb, 256);
          items += (int64_t)g.tiles_m * g.tiles_n;
          for (int pl = 0; pl < planes; ++pl) {
            void *out = P.kh ? (void *)((__half *)h->K + pl * P.kelems + b.koff) : (void *)(h->K + b.koff);
            if (tc3_encode_out_map(&maps[r * planes + pl], out, b.rows, b.ldb, b.ldb, P.kh))
              return fail(KKM_ECUDA, "%s", tc_gemm_error());
          }
        }
        T2Region *gregs = (T2Region *)((uint8_t *)h->ws + P.o_gregs);
        CUtensorMap *gmaps = (CUtensorMap *)((uint8_t *)h->ws + P.o_gmaps);
        CK(cudaMemcpyAsync(gregs, regs.data(), regs.size() * sizeof(T2Region), cudaMemcpyHostToDevice, h->st));
        CK(cudaMemcpyAsync(gmaps, maps.data(), maps.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice, h->st));
        if (tc3_gemm_launch_multi(h->tc, h->Xhi, h->Xlo, P.fp16, h->rscale, P.npad, P.dp, P.n, gregs,
                                  (int)regs.size(), items, gmaps, h->norms, h->kp, P.kh ? h->kscale : 0.f, planes,
                                  h->st, &h->launches, h->chain_kb)) {
          h->poisoned = true;
          return fail(KKM_ECUDA, "tcgen05 GEMM launch failed: %s", tc_gemm_error());
        }
        CK(cudaStreamSynchronize(h->st));  // (host copies of the regions and maps go out of scope)
      } else {
        for (const SymBand &b : P.bands) {
          const int64_t j0 = (int64_t)b.band * SYM_TB, i0 = j0 + b.row0;  // rows of the piece, columns >= band start
          CKR(launch_gemm(h, i0, b.rows, j0, b.ldb, h->K + b.koff, b.ldb));
        }
      }
    } else if (P.materialize) {
      CKR(launch_gemm(h, P.a0, P.nA, P.b0, P.ldk, h->K, P.ldk));
    }
    if (!evs.record(h->st)) return fail(KKM_ECUDA, "cudaEventCreate/Record failed");
    CK(cudaStreamSynchronize(h->st));
    if (h->p.timing) {
      float a = 0, b = 0;
      CK(cudaEventElapsedTime(&a, evs.v[0], evs.v[1]));
      CK(cudaEventElapsedTime(&b, evs.v[1], evs.v[2]));
      h->phase_ms[KKM_PH_INIT_PREP] += a;
      h->phase_ms[KKM_PH_INIT_GEMM] += b;
    }
    return KKM_OK;
  }();
  if (rc == KKM_OK && P.pr > 1) {  // process-column communicator: ranks gi + gj * pr, key gi
    ncclResult_t r = ncclCommSplit(h->comm, P.gj, P.gi, &h->colcomm, nullptr);
    if (r != ncclSuccess) rc = fail(KKM_ENCCL, "ncclCommSplit: %s", ncclGetErrorString(r));
    // one reduce-scatter of the real size now, so the communicator's connection setup is part
    // of the one-time init and not of the first iterations
    if (rc == KKM_OK) {
      cudaMemsetAsync(h->Scol, 0, (size_t)P.nApad * P.k * 8, h->st);
      r = ncclReduceScatter(h->Scol, h->Smine, (size_t)P.B * P.k, ncclDouble, ncclSum, h->colcomm, h->st);
      if (r != ncclSuccess) rc = fail(KKM_ENCCL, "ncclReduceScatter (warm-up): %s", ncclGetErrorString(r));
      else if (cudaStreamSynchronize(h->st) != cudaSuccess) rc = fail(KKM_ECUDA, "warm-up sync failed");
    }
  }
  // (p2p needs the a3 that reads the int64 S itself: a3fix; the single-CTA fused path reads fp64 S)
  // Opt-in (KKM_P2P=1): measured only 2 % faster than the NCCL allreduce at 4 GPUs, and
  // every rank reads all (P - 1) peers' whole S, so it is limited to P <= KKM_P2P_MAX_RANKS (4).
  // The decision is agreed by all ranks (an allreduce of the local wish) before the collective
  // setup, so ranks with different environments cannot issue mismatched collectives.
  if (rc == KKM_OK && P.a3fix && P.repl && P.nranks > 1) {
    int p2p_max = 4;
    if (const char *e = std::getenv("KKM_P2P_MAX_RANKS")) p2p_max = std::atoi(e);
    const char *want_env = std::getenv("KKM_P2P");
    int want = (want_env && std::atoi(want_env) == 1 && P.nranks <= p2p_max) ? 1 : 0;
    double tmo = 600.0;  // seconds a finalize waits for a peer's flag before it reports a timeout
    if (const char *e = std::getenv("KKM_P2P_TIMEOUT_S")) tmo = std::max(1.0, std::atof(e));
    h->p2p_timeout_ns = (unsigned long long)(tmo * 1e9);
    rc = agree_min(h, &want);
    if (rc == KKM_OK && want) rc = setup_p2p(h);
  }
  if (rc) {
    delete h;
    return rc;
  }
  *out = h;
  return KKM_OK;
}

int kkm_fit(kkm_handle h, int32_t *iters_run, double *J_trace, int64_t *changed) {
  if (!h) return fail(KKM_EINVAL, "handle is NULL");
  if (h->poisoned) return fail(KKM_ESTATE, "handle is poisoned by an earlier CUDA/NCCL error");
  const Plan &P = h->P;
  const int T = h->p.max_iter;
  EventList ev;  // 5 per iteration (timing mode)
  const bool timing = h->p.timing != 0;
  auto rec = [&](EventList &l) -> int {
    if (!l.record(h->st)) {
      h->poisoned = true;
      return fail(KKM_ECUDA, "cudaEventCreate/Record failed");
    }
    return KKM_OK;
  };
  h->a2ev.clear();
  int t = 0;
  h->time_a2 = timing;
  for (t = 0; t < T; ++t) {
    if (timing) CKR(rec(ev));
    const double *S = nullptr;
    int ns = 0;
    int64_t rows_pad = P.s_rows_pad;
    if (P.inc && h->s_valid) {  // f3: S of the current labels maintained incrementally
      S = h->Sinc;
      ns = 1;
      rows_pad = P.B;
    } else {
      CKR(launch_spmm(h, h->lab[h->cur], &S, &ns));  // a2 (+ 1.5D reduce-scatter)
      if (P.inc && P.nloc > 0) {
        sinc_set_kernel<<<(unsigned)ceil_div(P.nloc * P.k, 256), 256, 0, h->st>>>(S, ns, rows_pad, P.nloc, P.k,
                                                                                   h->Sinc);
        CKL();
      }
    }
    if (timing) CKR(rec(ev));
    if (P.fused) {  // a3 + a4 in one launch (the phase split is reported as a3)
      fused_update_kernel<<<1, FUSED_THREADS, (size_t)(P.k + 1) * FUSED_THREADS * 8 + P.k * 8, h->st>>>(
          S, ns, P.n, rows_pad, P.k, h->sizes[h->cur], h->lab[h->cur], h->diag, h->E, h->cnorm, h->J + t, 1,
          h->lab[h->cur ^ 1], h->sizes[h->cur ^ 1], h->changed + t, h->Dfull);
      CKL();
      if (timing) CKR(rec(ev));
    } else {
      CKR(run_cnorm(h, S, ns, rows_pad, h->E, h->cnorm, h->J + t, h->sizes[h->cur ^ 1], h->changed + t));  // a3
      if (timing) CKR(rec(ev));
      CKR(run_assign(h, h->changed + t));                                   // a4
    }
    if (timing) CKR(rec(ev));
    unsigned long long c = 1;
    if (h->p.stop_on_no_change || P.inc) {
      CK(cudaMemcpyAsync(&c, h->changed + t, 8, cudaMemcpyDeviceToHost, h->st));
      CK(cudaStreamSynchronize(h->st));
    }
    if (P.inc) {  // S for the new labels: unchanged, by the moved points, or a full pass next time
      if (c > 0 && (int64_t)c <= P.dmax) {
        CKR(delta_update(h, (int64_t)c));
        h->s_valid = true;
      } else {
        h->s_valid = c == 0;
      }
    }
    if (timing) CKR(rec(ev));
    h->cur ^= 1;
    h->have_last = true;
    if (h->p.stop_on_no_change && c == 0) {
      ++t;
      break;
    }
  }
  h->time_a2 = false;
  // J of the final labels (one more a2 + a3 pass, as the oracle's J_trace[iters])
  {
    const double *S = nullptr;
    int ns = 0;
    int64_t rows_pad = P.s_rows_pad;
    if (P.inc && h->s_valid) {
      S = h->Sinc;
      ns = 1;
      rows_pad = P.B;
    } else {
      CKR(launch_spmm(h, h->lab[h->cur], &S, &ns));
    }
    CKR(run_cnorm(h, S, ns, rows_pad, h->E2, h->cnorm2, h->J + t, nullptr, nullptr));
    h->cnorm2_valid = true;
  }
  std::vector<double> J((size_t)t + 1);
  std::vector<unsigned long long> ch((size_t)std::max(t, 1));
  CK(cudaMemcpyAsync(J.data(), h->J, (size_t)(t + 1) * 8, cudaMemcpyDeviceToHost, h->st));
  if (t > 0) CK(cudaMemcpyAsync(ch.data(), h->changed, (size_t)t * 8, cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  CKR(check_p2p(h));
  if (timing) {
    const std::vector<cudaEvent_t> &e5 = ev.v;
    for (size_t i = 0; i + 4 < e5.size(); i += 5) {  // the a2 phase includes the f3 S update
      float a, b, c, d;
      CK(cudaEventElapsedTime(&a, e5[i], e5[i + 1]));
      CK(cudaEventElapsedTime(&b, e5[i + 1], e5[i + 2]));
      CK(cudaEventElapsedTime(&c, e5[i + 2], e5[i + 3]));
      CK(cudaEventElapsedTime(&d, e5[i + 3], e5[i + 4]));
      h->phase_ms[KKM_PH_SPMM] += a + d;
      h->phase_ms[KKM_PH_CNORM] += b;
      h->phase_ms[KKM_PH_ASSIGN] += c;
    }
    const std::vector<cudaEvent_t> &a2 = h->a2ev.v;
    for (size_t i = 0; i + 1 < a2.size(); i += 2) {
      float a = 0;
      CK(cudaEventElapsedTime(&a, a2[i], a2[i + 1]));
      h->phase_ms[KKM_PH_A2_KERNEL] += a;
    }
  }
  h->a2ev.clear();
  if (iters_run) *iters_run = t;
  if (J_trace) std::memcpy(J_trace, J.data(), (size_t)(t + 1) * 8);
  if (changed)
    for (int i = 0; i < t; ++i) changed[i] = (int64_t)ch[i];
  (void)P;
  return KKM_OK;
}

int kkm_assign(kkm_handle h, int32_t *labels_out) {
  if (!h || !labels_out) return fail(KKM_EINVAL, "NULL argument");
  if (h->poisoned) return fail(KKM_ESTATE, "handle is poisoned");
  CKR(copy_any(h, labels_out, h->lab[h->cur], (size_t)h->P.n * 4));
  CK(cudaStreamSynchronize(h->st));
  return KKM_OK;
}

int kkm_objective(kkm_handle h, double *J) {
  if (!h || !J) return fail(KKM_EINVAL, "NULL argument");
  if (h->poisoned) return fail(KKM_ESTATE, "handle is poisoned");
  double *slot = h->J + h->P.max_iter + 1;
  const double *S = nullptr;
  int ns = 0;
  CKR(launch_spmm(h, h->lab[h->cur], &S, &ns));
  CKR(run_cnorm(h, S, ns, h->P.s_rows_pad, h->E2, h->cnorm2, slot, nullptr, nullptr));
  h->cnorm2_valid = true;
  CK(cudaMemcpyAsync(J, slot, 8, cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  CKR(check_p2p(h));
  return KKM_OK;
}

int kkm_set_labels(kkm_handle h, const int32_t *labels) {
  if (!h || !labels) return fail(KKM_EINVAL, "NULL argument");
  if (h->poisoned) return fail(KKM_ESTATE, "handle is poisoned");
  const Plan &P = h->P;
  // validated in the scratch buffer first: a rejected call leaves the current labels untouched
  int32_t *dst = h->lab[h->cur], *tmp = h->lab[h->cur ^ 1];
  CK(cudaMemsetAsync(h->bad, 0, 4, h->st));
  CK(cudaMemcpyAsync(tmp, labels, (size_t)P.n * 4, cudaMemcpyDefault, h->st));
  check_labels_kernel<<<(unsigned)ceil_div(P.n, 256), 256, 0, h->st>>>(tmp, P.n, P.k, h->bad);
  CKL();
  int bad = 0;
  CK(cudaMemcpyAsync(&bad, h->bad, 4, cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  if (!bad) {
    load_labels_kernel<<<(unsigned)ceil_div(P.lablen, 256), 256, 0, h->st>>>(tmp, dst, P.n, P.lablen, P.k, h->bad);
    CKL();
    CK(cudaMemsetAsync(h->sizes[h->cur], 0, (size_t)P.k * 4, h->st));
    histogram_kernel<<<std::min<int64_t>(ceil_div(P.n, 256), 1024), 256, (size_t)P.k * 4, h->st>>>(
        dst, P.n, P.k, h->sizes[h->cur]);
    CKL();
  }
  round_robin_kernel<<<(unsigned)ceil_div(P.lablen, 256), 256, 0, h->st>>>(tmp, P.n, P.lablen, P.k);
  CKL();
  CK(cudaStreamSynchronize(h->st));
  if (bad) return fail(KKM_ELABEL, "%d labels outside [0, %d); current labels kept", bad, P.k);
  h->have_last = false;
  h->cnorm2_valid = false;
  h->s_valid = false;
  return KKM_OK;
}

}  // extern "C"

namespace {

// Layout of kkm_predict's scratch: Y operands, sort scratch, sorted X (materialised handles
// only: streaming handles lend their own), the partials and the outputs.
struct PredictPlan {
  int64_t mpad;
  int splits, nblk;
  bool own_sorted;
  size_t oYf, oYhi, oYlo, oYn, oYr, oYd, oSp, oSx, oFx, oLab, oD, oPerm, oPos, oSeg, oBc, oBo, oShi, oSlo, oSn, oSr,
      total;
};

PredictPlan predict_plan(const kkm_ctx *h, int64_t m) {
  const Plan &P = h->P;
  PredictPlan q;
  q.mpad = round_up(std::max<int64_t>(m, 1), 256);
  q.nblk = (int)ceil_div(P.n, SORT_BLOCK);
  const int64_t tiles_n = ceil_div(P.n, 256);
  q.splits = (int)std::max<int64_t>(ceil_div(tiles_n, 512), ts_choose_splits((m + 1) / 2, P.n, h->num_sms / 2));
  q.own_sorted = P.materialize;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += (bytes + 255) / 256 * 256;
    return o;
  };
  const int k = P.k;
  q.oYf = take((size_t)q.mpad * P.ldf * 4);
  q.oYhi = take((size_t)q.mpad * P.dp * 2);
  q.oYlo = take((size_t)q.mpad * P.dp * 2);
  q.oYn = take((size_t)q.mpad * 4);
  q.oYr = take((size_t)q.mpad * 4);
  q.oYd = take((size_t)q.mpad * 8);
  q.oSp = take((size_t)q.mpad * k * 8);
  q.oSx = take((size_t)q.mpad * k * 8);
  q.oFx = take(16);
  q.oLab = take((size_t)q.mpad * 4);
  q.oD = take((size_t)q.mpad * k * 8);
  q.oPerm = take((size_t)P.lablen * 4);
  q.oPos = take((size_t)P.lablen * 4);
  q.oSeg = take((size_t)(k + 1) * 4);
  q.oBc = take((size_t)q.nblk * k * 4);
  q.oBo = take((size_t)q.nblk * k * 4);
  q.oShi = q.own_sorted ? take((size_t)P.npad * P.dp * 2) : 0;
  q.oSlo = q.own_sorted ? take((size_t)P.npad * P.dp * 2) : 0;
  q.oSn = q.own_sorted ? take((size_t)P.npad * 4) : 0;
  q.oSr = q.own_sorted ? take((size_t)P.npad * 4) : 0;
  q.total = off;
  return q;
}

int predict_run(kkm_ctx *h, const PredictPlan &q, uint8_t *t, const float *Y, int64_t m, int64_t ldy,
                int32_t *labels_out, double *D_out) {
  const Plan &P = h->P;
  const int k = P.k;
  float *Yf = (float *)(t + q.oYf), *yn = (float *)(t + q.oYn), *yr = (float *)(t + q.oYr);
  uint16_t *Yhi = (uint16_t *)(t + q.oYhi), *Ylo = (uint16_t *)(t + q.oYlo);
  double *yd = (double *)(t + q.oYd), *Sp = (double *)(t + q.oSp), *Dy = D_out ? (double *)(t + q.oD) : nullptr;
  int32_t *ylab = (int32_t *)(t + q.oLab);
  const bool own = q.own_sorted;
  SortedSet B{own ? (uint16_t *)(t + q.oShi) : h->Shi, own ? (uint16_t *)(t + q.oSlo) : h->Slo,
              own ? (float *)(t + q.oSn) : h->snorms, own ? (float *)(t + q.oSr) : h->srscale,
              (int32_t *)(t + q.oPerm), (int32_t *)(t + q.oPos), (int32_t *)(t + q.oSeg), (int32_t *)(t + q.oBc),
              (int32_t *)(t + q.oBo)};
  // a5 for the new points: split operands, norms, kappa(y, y) (prep_rows and diag read only
  // rows < m and columns < d of Yf, and write the split's pad rows/columns as zeros)
  CK(cudaMemcpy2DAsync(Yf, P.ldf * 4, Y, ldy * 4, P.d * 4, m, cudaMemcpyDefault, h->st));
  if (h->p.kind == KKM_KERNEL_GAUSSIAN) {  // the training points were centered (kkm_init)
    center_rows_kernel<<<(unsigned)ceil_div(m, 8), 256, 0, h->st>>>(Yf, P.ldf, m, P.d, h->mean);
    CKL();
  }
  prep_rows_kernel<<<(unsigned)ceil_div(q.mpad, 8), 256, 0, h->st>>>(Yf, P.ldf, m, q.mpad, P.d, yn, Yhi, Ylo, P.dp,
                                                                     P.fp16 ? 2 : 1, yr);
  CKL();
  if (h->p.kind == KKM_KERNEL_GAUSSIAN) {  // the tensor core's own y . y, as the training norms (kkm_init)
    TcGemm gy;
    if (tc3_self_dots(gy, Yhi, Ylo, P.fp16, yr, q.mpad, P.dp, m, yn, h->st, &h->launches, h->chain_kb)) {
      h->poisoned = true;
      return fail(KKM_ECUDA, "tensor-core self dots failed: %s", tc_gemm_error());
    }
  }
  diag_kernel<<<(unsigned)ceil_div(m, 8), 256, 0, h->st>>>(Yf, P.ldf, P.d, 0, m, h->p.kind, h->p.gamma, h->p.coef0,
                                                            h->p.degree, yd);
  CKL();
  // B = all n training points sorted by their current labels; A = Y
  CKR(sort_gather(h, h->lab[h->cur], 0, P.n, P.npad, B));
  TcStream &ts = h->ts_predict;
  const StreamA A{Yhi, Ylo, yn, yr, q.mpad, 0, m, q.mpad};
  // fixed-point scale of the streaming sums: n max|K(y, x)| 2^s < 2^61, |K(y, x)| <= max(K(y, y), K(x, x))
  double kmax = 1.0;
  if (h->p.kind != KKM_KERNEL_GAUSSIAN) {
    float *fm = (float *)(t + q.oFx);
    max_norm_kernel<<<1, 1024, 0, h->st>>>(h->norms, P.n, fm);
    CKL();
    max_norm_kernel<<<1, 1024, 0, h->st>>>(yn, m, fm + 1);
    CKL();
    float mx[2] = {0.f, 0.f};
    CK(cudaMemcpyAsync(mx, fm, 8, cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    const double nm = std::max((double)mx[0], (double)mx[1]);
    kmax = h->p.kind == KKM_KERNEL_LINEAR ? std::max(1e-30, nm)
                                          : std::pow(h->p.gamma * nm + std::fabs(h->p.coef0), (double)h->p.degree);
  }
  const double fx = std::ldexp(1.0, (int)std::floor(61.0 - std::log2(std::max(1e-300, (double)P.n * kmax * 1.0001))));
  CKR(stream_pass(h, ts, A, B, P.npad, P.n, 0, nullptr, 0, q.splits, fx, (long long *)(t + q.oSx), Sp));
  predict_kernel<<<(unsigned)ceil_div(m, 256), 256, 0, h->st>>>(Sp, 1, m, q.mpad, k, h->sizes[h->cur],
                                                                h->cnorm2, yd, ylab, Dy);
  CKL();
  CKR(copy_any(h, labels_out, ylab, (size_t)m * 4));
  if (D_out) CKR(copy_any(h, D_out, Dy, (size_t)m * k * 8));
  CK(cudaStreamSynchronize(h->st));
  return KKM_OK;
}

}  // namespace

extern "C" {

int kkm_predict_workspace_size(kkm_handle h, int64_t m, size_t *bytes) {
  if (!h || !bytes) return fail(KKM_EINVAL, "NULL argument");
  if (m < 0) return fail(KKM_EINVAL, "m=%lld < 0", (long long)m);
  *bytes = predict_plan(h, m).total;
  return KKM_OK;
}

int kkm_predict(kkm_handle h, const float *Y, int64_t m, int64_t ldy, int32_t *labels_out, double *D_out,
                void *workspace, size_t ws_bytes) {
  if (!h) return fail(KKM_EINVAL, "handle is NULL");
  if (h->poisoned) return fail(KKM_ESTATE, "handle is poisoned");
  const Plan &P = h->P;
  if (m < 0) return fail(KKM_EINVAL, "m=%lld < 0", (long long)m);
  if (m == 0) return KKM_OK;
  if (!Y || !labels_out) return fail(KKM_EINVAL, "NULL argument");
  if (ldy < P.d) return fail(KKM_EINVAL, "ldy=%lld < d=%lld", (long long)ldy, (long long)P.d);
  if (!P.tc) return fail(KKM_EUNSUP, "kkm_predict needs a tensor-core precision (FP16X3 or BF16X3)");
  const PredictPlan q = predict_plan(h, m);
  if (workspace) {
    if (((uintptr_t)workspace) & 255) return fail(KKM_EINVAL, "workspace must be 256-byte aligned");
    if (ws_bytes < q.total) return fail(KKM_ENOMEM, "workspace %zu bytes < required %zu", ws_bytes, q.total);
  }
  if (!h->cnorm2_valid) {  // c of the current labels: the kkm_objective pass (collective for nranks > 1)
    if (P.nranks > 1) return fail(KKM_ESTATE, "call kkm_fit or kkm_objective on every rank before kkm_predict");
    double J = 0.0;
    CKR(kkm_objective(h, &J));
  }
  if (workspace) return predict_run(h, q, (uint8_t *)workspace, Y, m, ldy, labels_out, D_out);
  uint8_t *t = nullptr;
  if (cudaMallocAsync((void **)&t, q.total, h->st) != cudaSuccess) {
    cudaGetLastError();
    return fail(KKM_ENOMEM, "kkm_predict: cannot allocate %zu temporary bytes", q.total);
  }
  const int rc = predict_run(h, q, t, Y, m, ldy, labels_out, D_out);
  cudaFreeAsync(t, h->st);
  if (rc == KKM_OK) CK(cudaStreamSynchronize(h->st));
  return rc;
}

int kkm_seed_kmeanspp(kkm_handle h, const double *u, int64_t *centers_out) {
  if (!h || !u) return fail(KKM_EINVAL, "NULL argument");
  if (h->poisoned) return fail(KKM_ESTATE, "handle is poisoned");
  const Plan &P = h->P;
  const int k = P.k;
  for (int t = 0; t < k; ++t)
    if (!(u[t] >= 0.0 && u[t] < 1.0)) return fail(KKM_EINVAL, "u[%d] = %g outside [0, 1)", t, u[t]);
  int64_t c0 = (int64_t)(u[0] * (double)P.n);
  if (c0 >= P.n) c0 = P.n - 1;
  uint8_t *t0 = nullptr;
  const size_t oD = 0, oL = round_up((int64_t)P.n * 8, 256), oC = oL + round_up((int64_t)P.n * 4, 256),
               total = oC + round_up((int64_t)k * 8, 256);
  if (cudaMallocAsync((void **)&t0, total, h->st) != cudaSuccess) {
    cudaGetLastError();
    return fail(KKM_ENOMEM, "kkm_seed_kmeanspp: cannot allocate %zu temporary bytes", total);
  }
  double *D = (double *)(t0 + oD);
  int32_t *lab = (int32_t *)(t0 + oL);
  int64_t *cen = (int64_t *)(t0 + oC);
  int rc = [&]() -> int {
    CK(cudaMemcpyAsync(cen, &c0, 8, cudaMemcpyHostToDevice, h->st));
    for (int t = 0; t < k; ++t) {
      kpp_dist_kernel<<<(unsigned)ceil_div(P.n, 8), 256, 0, h->st>>>(h->Xf, P.ldf, P.n, P.d, cen, t, h->p.kind,
                                                                      h->p.gamma, h->p.coef0, h->p.degree, D, lab);
      CKL();
      if (t + 1 < k) {
        kpp_pick_kernel<<<1, 1024, 0, h->st>>>(D, P.n, u[t + 1], t, cen);
        CKL();
      }
    }
    if (centers_out) CKR(copy_any(h, centers_out, cen, (size_t)k * 8));
    CK(cudaStreamSynchronize(h->st));
    return kkm_set_labels(h, lab);  // validates, sets sizes, invalidates the derived state
  }();
  cudaFreeAsync(t0, h->st);
  cudaStreamSynchronize(h->st);
  return rc;
}

int kkm_debug_read(kkm_handle h, int32_t what, void *dst) {
  if (!h || !dst) return fail(KKM_EINVAL, "NULL argument");
  if (h->poisoned) return fail(KKM_ESTATE, "handle is poisoned");
  const Plan &P = h->P;
  const int prev = h->cur ^ 1;  // buffers of the labels entering the last iteration
  switch (what) {
    case KKM_DBG_E: CKR(copy_any(h, dst, h->E + (P.row0 - P.a_row0) * P.k, (size_t)P.nloc * P.k * 8)); break;
    case KKM_DBG_CNORM: CKR(copy_any(h, dst, h->cnorm, (size_t)P.k * 8)); break;
    case KKM_DBG_SIZES:
      CKR(copy_any(h, dst, h->sizes[h->have_last ? prev : h->cur], (size_t)P.k * 4));
      break;
    case KKM_DBG_DIAG: CKR(copy_any(h, dst, h->diag + (P.row0 - P.a_row0), (size_t)P.nloc * 8)); break;
    case KKM_DBG_DFULL:
      CKR(copy_any(h, dst, h->Dfull + (P.row0 - P.a_row0) * P.k, (size_t)P.nloc * P.k * 8));
      break;
    case KKM_DBG_LABELS_PREV:
      CKR(copy_any(h, dst, h->lab[h->have_last ? prev : h->cur], (size_t)P.n * 4));
      break;
    default: return fail(KKM_EINVAL, "unknown debug selector %d", what);
  }
  CK(cudaStreamSynchronize(h->st));
  return KKM_OK;
}

int kkm_stored_k_row(kkm_handle h, int64_t i, double *dst) {
  if (!h || !dst) return fail(KKM_EINVAL, "NULL argument");
  if (h->poisoned) return fail(KKM_ESTATE, "handle is poisoned");
  const Plan &P = h->P;
  if (i < 0 || i >= P.n) return fail(KKM_EINVAL, "row %lld out of range", (long long)i);
  if (!P.materialize) return fail(KKM_ESTATE, "the handle streams K: nothing is stored");
  std::vector<double> out((size_t)P.n, std::nan(""));
  if (P.sym) {
    const SymBand *piece = nullptr;
    for (const SymBand &b : P.bands) {
      const int64_t r0 = (int64_t)b.band * SYM_TB + b.row0;
      if (i >= r0 && i < r0 + b.rows) piece = &b;
    }
    if (!piece) return fail(KKM_ESTATE, "row %lld is not stored on this rank", (long long)i);
    const int64_t j0 = (int64_t)piece->band * SYM_TB;
    const int64_t r = i - j0 - piece->row0, cols = P.n - j0;
    if (P.kh) {
      std::vector<__half> hi((size_t)cols), lo((size_t)cols);
      const __half *base = (const __half *)h->K + piece->koff + r * piece->ldb;
      CK(cudaMemcpyAsync(hi.data(), base, (size_t)cols * 2, cudaMemcpyDeviceToHost, h->st));
      if (P.kplanes > 1)
        CK(cudaMemcpyAsync(lo.data(), base + P.kelems, (size_t)cols * 2, cudaMemcpyDeviceToHost, h->st));
      CK(cudaStreamSynchronize(h->st));
      const double inv = 1.0 / (double)h->kscale;
      for (int64_t j = 0; j < cols; ++j)
        out[(size_t)(j0 + j)] = ((double)__half2float(hi[(size_t)j]) +
                                 (P.kplanes > 1 ? (double)__half2float(lo[(size_t)j]) : 0.0)) * inv;
    } else {
      std::vector<float> v((size_t)cols);
      CK(cudaMemcpyAsync(v.data(), h->K + piece->koff + r * piece->ldb, (size_t)cols * 4, cudaMemcpyDeviceToHost,
                         h->st));
      CK(cudaStreamSynchronize(h->st));
      for (int64_t j = 0; j < cols; ++j) out[(size_t)(j0 + j)] = v[(size_t)j];
    }
  } else {  // full K rows: the A set's rows x the B set's columns
    if (i < P.a0 || i >= P.a0 + P.nA) return fail(KKM_ESTATE, "row %lld is not stored on this rank", (long long)i);
    std::vector<float> v((size_t)P.nB);
    CK(cudaMemcpyAsync(v.data(), h->K + (i - P.a0) * P.ldk, (size_t)P.nB * 4, cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    for (int64_t j = 0; j < P.nB; ++j) out[(size_t)(P.b0 + j)] = v[(size_t)j];
  }
  std::memcpy(dst, out.data(), (size_t)P.n * 8);
  return KKM_OK;
}

int kkm_kernel_tile(kkm_handle h, int64_t i0, int64_t j0, int32_t m, int32_t nc, float *dst) {
  if (!h || !dst) return fail(KKM_EINVAL, "NULL argument");
  if (h->poisoned) return fail(KKM_ESTATE, "handle is poisoned");
  const Plan &P = h->P;
  if (m < 1 || nc < 1 || i0 < 0 || j0 < 0 || i0 + m > P.n || j0 + nc > P.n)
    return fail(KKM_EINVAL, "tile out of range");
  float *tmp = nullptr;
  const int64_t ldt = round_up(nc, 4);  // TMA-store pitch
  CK(cudaMallocAsync((void **)&tmp, (size_t)m * ldt * 4, h->st));
  int rc = launch_gemm(h, i0, m, j0, nc, tmp, ldt);
  if (rc == KKM_OK) {
    cudaError_t e = cudaMemcpy2DAsync(dst, (size_t)nc * 4, tmp, (size_t)ldt * 4, (size_t)nc * 4, m,
                                      cudaMemcpyDefault, h->st);
    if (e != cudaSuccess) rc = fail(KKM_ECUDA, "kernel_tile copy: %s", cudaGetErrorString(e));
  }
  cudaFreeAsync(tmp, h->st);
  if (rc) return rc;
  CK(cudaStreamSynchronize(h->st));
  return KKM_OK;
}

int kkm_phase_ms(kkm_handle h, float *ms) {
  if (!h || !ms) return fail(KKM_EINVAL, "NULL argument");
  std::memcpy(ms, h->phase_ms, sizeof(h->phase_ms));
  return KKM_OK;
}

int kkm_launch_count(kkm_handle h, int64_t *count) {
  if (!h || !count) return fail(KKM_EINVAL, "NULL argument");
  *count = h->launches;
  return KKM_OK;
}

int kkm_destroy(kkm_handle h) {
  if (!h) return KKM_OK;
  cudaStreamSynchronize(h->st);
  if (h->xbuf) {
    // no rank frees its exchange buffer while a peer may still read it: raise the own flag to
    // DONE (after the stream is idle) and wait, bounded, for every peer's DONE -- no NCCL here, so
    // destroy stays safe after the communicator is gone or when handles die in any order
    const unsigned long long done = ~0ull;
    cudaMemcpy(h->xbuf + h->xflag_off, &done, 8, cudaMemcpyHostToDevice);
    const auto t0 = std::chrono::steady_clock::now();
    bool all_done = true;
    for (void *q : h->xpeers) {
      unsigned long long v = 0;
      while (cudaMemcpy(&v, (uint8_t *)q + h->xflag_off, 8, cudaMemcpyDeviceToHost) == cudaSuccess && v != done &&
             std::chrono::steady_clock::now() - t0 < std::chrono::seconds(20))
        std::this_thread::sleep_for(std::chrono::microseconds(200));
      all_done = all_done && v == done;
    }
    for (void *q : h->xpeers) cudaIpcCloseMemHandle(q);
    // a peer that never reported DONE may still read this buffer: keep it (leak) rather than free
    if (all_done) cudaFree(h->xbuf);
    cudaGetLastError();
  }
  if (h->colcomm) ncclCommDestroy(h->colcomm);
  delete h;
  return KKM_OK;
}

int kkm_get_unique_id(char id[128]) {
  if (!id) return fail(KKM_EINVAL, "id is NULL");
  ncclUniqueId u;
  ncclResult_t r = ncclGetUniqueId(&u);
  if (r != ncclSuccess) return fail(KKM_ENCCL, "ncclGetUniqueId: %s", ncclGetErrorString(r));
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  std::memcpy(id, &u, 128);
  return KKM_OK;
}

int kkm_comm_init(void **comm, int32_t nranks, int32_t rank, const char id[128]) {
  if (!comm || !id) return fail(KKM_EINVAL, "NULL argument");
  ncclUniqueId u;
  std::memcpy(&u, id, 128);
  ncclComm_t c;
  ncclResult_t r = ncclCommInitRank(&c, nranks, u, rank);
  if (r != ncclSuccess) return fail(KKM_ENCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
  *comm = c;
  return KKM_OK;
}

int kkm_comm_destroy(void *comm) {
  if (!comm) return KKM_OK;
  ncclResult_t r = ncclCommDestroy((ncclComm_t)comm);
  if (r != ncclSuccess) return fail(KKM_ENCCL, "ncclCommDestroy: %s", ncclGetErrorString(r));
  return KKM_OK;
}

}  // extern "C"
