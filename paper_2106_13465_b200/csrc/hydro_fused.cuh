// hydro_fused.cuh -- the FUSED schedule: one kernel per time step.
//
// Included by hydro_kernels.cu inside namespace hb { namespace { ... } } (so
// it is compiled in both arithmetics, like the split sweeps).
//
// One reference step (proj/src/schedulers.cpp:103-116) is a column sweep, an
// apply_boundary and a row sweep.  The split schedule runs them as two
// launches that each stream the whole state through HBM (read 32 B + write
// 32 B per cell per sweep: 128 B per cell-step).  sweep_xy_kernel does both
// sweeps in one pass over the state (64 B per cell-step): the column sweep's
// output U_b never leaves shared memory.
//
// Work item: a BAND of kFW = 120 output columns [j0, j0 + 119] (15 column
// blocks of the tiled layout) x a segment of grid rows.  The CTA's 4 warps:
//   * column phase -- the strip walker of the split sweeps (walk_strip), one
//     lane per column strip j0-2 .. j0+121 (124 strips: the row sweep's
//     stencil halo), streaming U_a down the rows through a TMA ring of 4-row
//     chunks {8 cols, 17 blocks, 4 rows, 4 vars} (17 KB, one load per chunk
//     for the CTA); each updated cell goes to a U_b row in shared memory
//     (a "slot" of 4 rows), the band's y-wall ghost columns (grid.cpp:44-59)
//     written by the lanes owning columns 1, 2, ny-1, ny;
//   * row phase -- once a 4-row chunk of U_b rows is complete (CTA barrier),
//     warp w sweeps row w of it LANE-PARALLEL: lane l holds the 4 adjacent
//     cells j0-4+4l .. j0-1+4l (lanes 1..30: the 120 outputs; lanes 0 and 31:
//     the halo), converts, reconstructs and solves its own 4 interfaces, and
//     gets the neighbour primitives, the right face of cell -1 and the flux
//     at its right edge by warp shuffles -- the same per-cell work as the
//     walker (one conversion, one predictor, one Riemann solve, one update).
//     The updated row goes back into its slot in place and leaves with TMA
//     bulk-tensor stores (one per variable), the x-wall ghost rows of the
//     next step (grid.cpp:26-42) with plain stores, the dt speeds into the
//     warp's maximum (compute_dt, euler_kernel.cpp:233-242).
// The arithmetic is the split sweeps' (the same physics functions, the same
// math policy), and every cell update is a pure function of its 5-cell
// window, so the results are bitwise those of the split schedule.  A work
// item whose fast pass left its proven range is redone by the whole CTA with
// the exact policy.  Uniform windows: the column walker keeps the split
// sweeps' uniform-window identity; a row whose 128 cells are bitwise equal to
// a state whose (uniform-window) update this warp already evaluated to the
// identity in this launch keeps its input (the same bits as evaluating it).
//
// The run's last step (last_step) leaves the reference's final ghost bands
// behind instead of the next step's: its last apply_boundary ran on the
// column-sweep output, so the x-wall ghost rows come from the row phase's
// inputs and the y-wall ghost columns from the slot (finish_kernel's job in
// the split schedule).
//
// Row slabs (PEER): the rows a neighbour's next column sweep needs are also
// stored into its inbox (peer memory), like the split row sweep does; the
// per-step exchange copies the own inbox into the ghost rows of whichever
// buffer holds the state.
//
// Exact-10 flux (FLUX 1): the same kernel with the exact solver at every
// interface (the column walker with its interface memo, the row phase
// without); whole domains only (slabs with the exact flux stay split).
//
// Not fused: one leading step of a run with an odd step count (the state
// ping-pongs between the two buffers and must end in the first).

// ---- layout -------------------------------------------------------------------
constexpr int kFStrips = kFW + 4;                 // column-phase strips j0-2 .. j0+121
constexpr int kFLoadCols = 8 * kFLoadBlocks;      // 136: loaded columns j0-8 .. j0+127
constexpr int kFNBA = 8;                          // U_a ring buffers (a power of two)
constexpr uint32_t kFRowBytesA = kFLoadCols * 8;  // 1088
constexpr uint32_t kFVarBytesA = 4 * kFRowBytesA; // 4352: [var][row][col]
constexpr uint32_t kFChunkBytes = 4 * kFVarBytesA;  // 17408
constexpr int kFPos = 144;                        // slot positions: column j at j - j0 + 16
constexpr uint32_t kFVarBytesS = kFPos * 8;       // 1152 (9 x 128)
constexpr uint32_t kFRowBytesS = 4 * kFVarBytesS; // 4608: [row][var][pos]
constexpr uint32_t kFSlotBytes = 4 * kFRowBytesS; // 18432
#ifndef HB_FNS
#define HB_FNS 4
#endif
#ifndef HB_FLAG
#define HB_FLAG 2
#endif
constexpr int kFNS = HB_FNS;                      // slots (chunks in hand-over)
// The row warps release the slot of chunk n - kFLag when they take chunk n:
// with kFLag = 2 the stores a row warp issued for chunk n - 1 need not have
// read their slot yet (cp.async.bulk.wait_group.read 1), so a warp never
// waits for the stores it has just issued.
constexpr int kFLag = HB_FLAG;
#ifndef HB_FONEBAR
#define HB_FONEBAR 1
#endif

static_assert(kFLag >= 1 && kFLag <= 2 && kFLag < kFNS, "slot release lag");
constexpr uint32_t kFSlotOff = kFNBA * kFChunkBytes;
constexpr uint32_t kFBarOff = kFSlotOff + kFNS * kFSlotBytes;
constexpr uint32_t kFHdrOff = kFBarOff + kFNBA * 8;
constexpr uint32_t kFFlagOff = kFHdrOff + kFNS * 32;
constexpr uint32_t kFUniOff = kFFlagOff + 16;       // per slot: FusedUni
constexpr uint32_t kFUniBytes = 160;
constexpr uint32_t kFEdgeOff = kFUniOff + kFNS * kFUniBytes;  // row warps' wall-band memos (EdgeMemo)
constexpr uint32_t kFEdgeBytes = 80;
constexpr uint32_t kFMemoOff = kFEdgeOff + 4 * 2 * kFEdgeBytes;  // exact-10: the column warps' memos
constexpr int kFSmemBytes = (int)kFMemoOff + 128;             // + alignment
constexpr int kFSmemBytesEx = kFSmemBytes + 13 * 1024;

// ---- warp shuffles of the row phase ------------------------------------------
__device__ __forceinline__ double shfl_up_d(double v) {
  return __hiloint2double(__shfl_up_sync(0xffffffffu, __double2hiint(v), 1),
                          __shfl_up_sync(0xffffffffu, __double2loint(v), 1));
}
__device__ __forceinline__ double shfl_dn_d(double v) {
  return __hiloint2double(__shfl_down_sync(0xffffffffu, __double2hiint(v), 1),
                          __shfl_down_sync(0xffffffffu, __double2loint(v), 1));
}
__device__ __forceinline__ double shfl_d(double v, int src) {
  return __hiloint2double(__shfl_sync(0xffffffffu, __double2hiint(v), src),
                          __shfl_sync(0xffffffffu, __double2loint(v), src));
}
__device__ __forceinline__ Prim shfl_up(const Prim& w) {
  return {shfl_up_d(w.r), shfl_up_d(w.va), shfl_up_d(w.vb), shfl_up_d(w.p)};
}
__device__ __forceinline__ Prim shfl_dn(const Prim& w) {
  return {shfl_dn_d(w.r), shfl_dn_d(w.va), shfl_dn_d(w.vb), shfl_dn_d(w.p)};
}
__device__ __forceinline__ Flux shfl_dn(const Flux& f) {
  return {shfl_dn_d(f.m), shfl_dn_d(f.ma), shfl_dn_d(f.mb), shfl_dn_d(f.e)};
}
__device__ __forceinline__ Cons shfl(const Cons& u, int src) {
  return {shfl_d(u.r, src), shfl_d(u.ma, src), shfl_d(u.mb, src), shfl_d(u.e, src)};
}
__device__ __forceinline__ Face shfl_up(const Face& f) {
  Face o;
  o.w = shfl_up(f.w);
  o.rr.b = o.w.r;  // every Face's reciprocal is of its own density (face_prim)
  o.rr.r = shfl_up_d(f.rr.r);
  o.rr.pos = __shfl_up_sync(0xffffffffu, (int)f.rr.pos, 1) != 0;
#ifdef HB_TOLERANCE
  o.ma = shfl_up_d(f.ma);
  o.mb = shfl_up_d(f.mb);
  o.e = shfl_up_d(f.e);
#endif
  return o;
}

// Per-warp memo of the row phase's uniform-row identity (this launch: one dt).
struct RowMemo {
  bool valid;
  Cons u;      // a state whose uniform-window row update was the identity
  double spd;  // its dt signal speed
};

// The same memo for the rows of a band at a y-wall, whose ghost columns hold
// the wall's image G of the interior state U (reflecting walls: the normal
// momentum negated, which differs from U even at rest: -0 against +0): a row
// with U in every interior column and G in every ghost column whose update
// this warp has already evaluated to the identity in this launch.  One per
// row warp and wall side, in shared memory.
struct EdgeMemo {
  double u[4], g[4];  // r, mom_y, mom_x, E (row orientation)
  double spd;
  double valid;
};
static_assert(sizeof(EdgeMemo) == kFEdgeBytes, "EdgeMemo layout");

// What a row contributes: the largest dt signal speed, the first errors (this
// step's, and the dt of the next step's), uniform-window updates taken.
struct RowAcc {
  double spd;
  unsigned long long ekey, dtkey;
  unsigned nskip;
  __device__ __forceinline__ void clear() {
    spd = 0.0;
    ekey = dtkey = kNoError;
    nskip = 0;
  }
  __device__ __forceinline__ void add(const RowAcc& o) {
    spd = smax(spd, o.spd);
    keep_min(ekey, o.ekey);
    keep_min(dtkey, o.dtkey);
    nskip += o.nskip;
  }
};

// Geometry of the row a warp sweeps (lane-parallel): lane l holds columns
// jb .. jb+3, jb = j0 - 4 + 4 l; valid cells j in [jlo, jhi] (the band's
// stencil halo inside the strip -1 .. ny+2), outputs j0 .. ohi on lanes 1..30.
struct RowGeo {
  int j0, jb, jlo, jhi, ohi;
  unsigned long long key_base, dt_base;
};

// The row sweep of one row's 4-cell lane blocks with math policy M: loop 1
// conversions, loop 2 predictor + faces, loop 3 HLLC, loop 4 update and the
// dt speed (euler_kernel.cpp:111-242), the neighbours' primitives, the right
// face of cell -1 and the flux at the lane's right edge by shuffles.  Results
// in out[] (outputs only), contributions in acc; returns false if the fast
// pass left its proven range on an output's stencil.
template <class M, int FLUX>
__device__ __forceinline__ bool row_eval(const Cons (&u)[4], const bool (&outk)[4], int lane,
                                         const RowGeo& rg, const Gas& g, double dtdx, RowAcc& acc,
                                         Cons (&out)[4], bool& ident, double& sp0) {
  M m;
  if constexpr (M::kFast) m.ok = g.fast;
  const double half = 0.5 * dtdx;
  Prim w[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int f = to_prim(m, u[k], g, w[k]);
    const int j = rg.jb + k;
    if (f >= 0 && j >= rg.jlo && j <= rg.jhi)
      keep_min(acc.ekey, rg.key_base | ((unsigned long long)(j + 1) << 2) | f);
  }
  const Prim wm1 = shfl_up(w[3]);  // cell -1 (lane - 1's cell 3)
  const Prim w4 = shfl_dn(w[0]);   // cell 4 (lane + 1's cell 0)
  Face fl0, frp;
  Flux F1, F2, F3;
  NoMemo nomemo{};
  // interface k lies between columns jb+k-1 and jb+k; a Riemann failure
  // (exact-10: vacuum, exact_riemann.cpp:55-57) counts where the interface
  // bounds an output cell of the band (strip cell of its left column: jb+k)
  auto rfail = [&](int k, int f) {
    const int jl = rg.jb + k - 1, jr = rg.jb + k;
    if (f >= 0 && ((jr >= rg.j0 && jr <= rg.ohi) || (jl >= rg.j0 && jl <= rg.ohi)))
      keep_min(acc.ekey, rg.key_base | (1ull << 20) | ((unsigned long long)(rg.jb + k) << 2) | f);
  };
  int fr_ = -1;
  {
    Cons el, er;
    predict_evolved(m, wm1, w[0], w[1], half, g, el, er);
    fl0 = face_prim(m, el, w[0], g);
    frp = face_prim(m, er, w[0], g);
  }
  {
    Cons el, er;
    predict_evolved(m, w[0], w[1], w[2], half, g, el, er);
    const Face fl = face_prim(m, el, w[1], g);
    F1 = riemann<FLUX>(m, frp, fl, g, fr_, nomemo);
    rfail(1, fr_);
    frp = face_prim(m, er, w[1], g);
  }
  {
    Cons el, er;
    predict_evolved(m, w[1], w[2], w[3], half, g, el, er);
    const Face fl = face_prim(m, el, w[2], g);
    F2 = riemann<FLUX>(m, frp, fl, g, fr_, nomemo);
    rfail(2, fr_);
    frp = face_prim(m, er, w[2], g);
  }
  {
    Cons el, er;
    predict_evolved(m, w[2], w[3], w4, half, g, el, er);
    const Face fl = face_prim(m, el, w[3], g);
    F3 = riemann<FLUX>(m, frp, fl, g, fr_, nomemo);
    rfail(3, fr_);
    frp = face_prim(m, er, w[3], g);
  }
  const Face frm1 = shfl_up(frp);  // right face of cell -1
  const Flux F0 = riemann<FLUX>(m, frm1, fl0, g, fr_, nomemo);
  rfail(0, fr_);
  const Flux F4 = shfl_dn(F0);     // flux through this lane's right edge
  // (lanes 0 and 31 carry only halo cells, but lane 1's first interface and
  // lane 30's last flux come from them -- clamped copies of valid cells where
  // their blocks leave the band's halo -- so their range flags count too)
  ident = true;
  sp0 = 0.0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const Flux& fl = k == 0 ? F0 : k == 1 ? F1 : k == 2 ? F2 : F3;
    const Flux& fr = k == 0 ? F1 : k == 1 ? F2 : k == 2 ? F3 : F4;
    M mu = m;
    if constexpr (M::kFast) mu.ok = true;
    Cons un = u[k];
    Recip rr;
    UpdAux aux;
    const int fU = update_cell(mu, un, fl, fr, dtdx, rr, aux);
    double sp;
    const int fD = dt_speed(mu, un, rr, aux, g, sp);
    out[k] = u[k];
    if (outk[k]) {
      const int j = rg.jb + k;
      if constexpr (M::kFast) m.ok = m.ok & mu.ok;
      if (fU >= 0)
        keep_min(acc.ekey, rg.key_base | (2ull << 20) | ((unsigned long long)(j + 1) << 2) | fU);
      if (fD >= 0) keep_min(acc.dtkey, rg.dt_base | ((unsigned long long)j << 2) | fD);
      else acc.spd = smax(acc.spd, sp);
      ident = ident & (fU < 0) & (fD < 0) & same_bits(un, u[k]);
      out[k] = un;
    }
    if (k == 0) sp0 = sp;
  }
  return m.ok;
}

// The row phase of one grid row: slot row at hb_smem offset `at` (U_b of
// columns j0-2 .. j0+121 at positions 14 .. 137), updated in place.  Row
// orientation (the row sweep's): mom_a = mom_y (var 2), mom_b = mom_x (var 1).
template <int FLUX>
__device__ __forceinline__ void fused_row(uint32_t at, int lane, const RowGeo& rg, int ny,
                                          const Gas& g, double dtdx, RowMemo& memo, EdgeMemo* edge,
                                          RowAcc& acc, Cons (&u)[4], Cons (&out)[4],
                                          bool (&outk)[4]) {
  {
    const uint8_t* p = hb_smem + at + (12 + 4 * lane) * 8;
    const double2 r01 = *(const double2*)(p), r23 = *(const double2*)(p + 16);
    const double2 x01 = *(const double2*)(p + kFVarBytesS), x23 = *(const double2*)(p + kFVarBytesS + 16);
    const double2 y01 = *(const double2*)(p + 2 * kFVarBytesS),
                  y23 = *(const double2*)(p + 2 * kFVarBytesS + 16);
    const double2 e01 = *(const double2*)(p + 3 * kFVarBytesS),
                  e23 = *(const double2*)(p + 3 * kFVarBytesS + 16);
    u[0] = {r01.x, y01.x, x01.x, e01.x};
    u[1] = {r01.y, y01.y, x01.y, e01.y};
    u[2] = {r23.x, y23.x, x23.x, e23.x};
    u[3] = {r23.y, y23.y, x23.y, e23.y};
  }
  // cells outside the strip or the band's halo hold no state: they take the
  // nearest valid cell (their results are discarded; the copies keep the
  // discarded arithmetic inside the valid states' ranges)
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int j = rg.jb + k;
    if (j < rg.jlo || j > rg.jhi) {
      const uint8_t* p = hb_smem + at + ((j < rg.jlo ? rg.jlo : rg.jhi) - rg.j0 + 16) * 8;
      u[k] = {*(const double*)p, *(const double*)(p + 2 * kFVarBytesS),
              *(const double*)(p + kFVarBytesS), *(const double*)(p + 3 * kFVarBytesS)};
    }
    outk[k] = (lane >= 1) & (lane <= 30) & (j <= rg.ohi);
  }
  // uniform row: every cell equals column j0's
  const Cons ref = shfl(u[0], 1);
  const bool uni = __all_sync(0xffffffffu, same_bits(u[0], ref) & same_bits(u[1], ref) &
                                               same_bits(u[2], ref) & same_bits(u[3], ref));
  if (uni && memo.valid && same_bits(memo.u, ref)) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      out[k] = u[k];
      if (outk[k]) ++acc.nskip;
    }
    acc.spd = smax(acc.spd, memo.spd);
    return;
  }
  // a band at a y-wall: U in the interior columns, the wall's image G in the
  // ghost columns (see EdgeMemo)
  const bool wall_l = rg.jlo < 1, wall_r = rg.jhi > ny;
  bool pat = false;
  Cons G = ref;
  EdgeMemo* const em = edge + (wall_l ? 0 : 1);
  if (!uni && (wall_l | wall_r)) {
    const uint8_t* pg = hb_smem + at + ((wall_l ? 0 : ny + 1) - rg.j0 + 16) * 8;
    G = {*(const double*)pg, *(const double*)(pg + 2 * kFVarBytesS), *(const double*)(pg + kFVarBytesS),
         *(const double*)(pg + 3 * kFVarBytesS)};
    bool okc = true;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      int j = rg.jb + k;
      j = j < rg.jlo ? rg.jlo : (j > rg.jhi ? rg.jhi : j);
      okc &= same_bits(u[k], (j < 1 || j > ny) ? G : ref);
    }
    pat = __all_sync(0xffffffffu, okc);
    if (pat && em->valid != 0.0 &&
        same_bits(Cons{em->u[0], em->u[1], em->u[2], em->u[3]}, ref) &&
        same_bits(Cons{em->g[0], em->g[1], em->g[2], em->g[3]}, G)) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        out[k] = u[k];
        if (outk[k]) ++acc.nskip;
      }
      acc.spd = smax(acc.spd, em->spd);
      return;
    }
  }
  RowAcc r;
  r.clear();
  bool ident;
  double sp0;
  const bool ok = row_eval<FastMath, FLUX>(u, outk, lane, rg, g, dtdx, r, out, ident, sp0);
  const bool fast = __all_sync(0xffffffffu, ok);
  if (!fast) {  // an operand left the fast pass's range: the row again, exactly
    r.clear();
    row_eval<ExactMath, FLUX>(u, outk, lane, rg, g, dtdx, r, out, ident, sp0);
  }
  acc.add(r);
  // write the outputs back in place
  uint8_t* p = hb_smem + at + (12 + 4 * lane) * 8;
  if (outk[0] & outk[3]) {
    *(double2*)(p) = make_double2(out[0].r, out[1].r);
    *(double2*)(p + 16) = make_double2(out[2].r, out[3].r);
    *(double2*)(p + kFVarBytesS) = make_double2(out[0].mb, out[1].mb);
    *(double2*)(p + kFVarBytesS + 16) = make_double2(out[2].mb, out[3].mb);
    *(double2*)(p + 2 * kFVarBytesS) = make_double2(out[0].ma, out[1].ma);
    *(double2*)(p + 2 * kFVarBytesS + 16) = make_double2(out[2].ma, out[3].ma);
    *(double2*)(p + 3 * kFVarBytesS) = make_double2(out[0].e, out[1].e);
    *(double2*)(p + 3 * kFVarBytesS + 16) = make_double2(out[2].e, out[3].e);
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (outk[k]) {
        double* q = (double*)(p + 8 * k);
        q[0] = out[k].r;
        q[kFPos] = out[k].mb;
        q[2 * kFPos] = out[k].ma;
        q[3 * kFPos] = out[k].e;
      }
  }
  // a uniform row whose update was the identity on every output: remember
  // the state for this launch
  const bool all_ident = __all_sync(0xffffffffu, ident);
  const double sp_ref = shfl_d(sp0, 1);
  if (uni && all_ident) {
    memo.valid = true;
    memo.u = ref;
    memo.spd = sp_ref;
  }
  if (pat && all_ident) {
    __syncwarp();
    if (lane == 0) {
      em->u[0] = ref.r; em->u[1] = ref.ma; em->u[2] = ref.mb; em->u[3] = ref.e;
      em->g[0] = G.r; em->g[1] = G.ma; em->g[2] = G.mb; em->g[3] = G.e;
      em->spd = sp_ref;
      em->valid = 1.0;
    }
    __syncwarp();
  }
}

// Named barriers of the column -> row hand-over (bar 0 is __syncthreads):
// FULL(s) = 1 + s (column warps arrive, row warps sync), EMPTY(s) = 1 + kFNS
// + s (row warps arrive, column warps sync), 1 + 2 kFNS = the column warps
// alone.
__device__ __forceinline__ void bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
constexpr int kFBarFull = 1, kFBarEmpty = 1 + kFNS, kFBarCol = 1 + 2 * kFNS;
static_assert(kFBarCol < 16, "named barriers");

// A published chunk's header (one per slot): which rows, of which pass.
struct FusedHdr {
  int tag;    // 2 x item sequence number + pass (0 fast, 1 exact redo)
  int i0;     // grid row of the slot's row 0
  int nrows;  // rows of the chunk inside the item (1..4)
  int j0;     // band's first output column
  int first;  // first chunk of its pass
  int end;    // no more chunks
  int pad[2];
};

// What the column warps know about a published chunk (one record per slot):
// uni[w] != 0 -- column warp w took the chunk as part of a steady uniform run
// (every cell of its 32 strips x 4 rows bitwise equal to st[w], updated by the
// identity), in a band without wall or inactive strips.  When all four agree
// on one state the chunk's rows are uniform rows of that state, and the row
// warps need not read them to know it.
struct FusedUni {
  int uni[4];
  int pad[4];
  double st[4][4];  // r, mom_x, mom_y, E (column orientation)
};
static_assert(sizeof(FusedUni) == kFUniBytes, "FusedUni layout");

__device__ __forceinline__ unsigned long long diff_bits(const Cons& a, const Cons& b) {
  return ((unsigned long long)__double_as_longlong(a.r) ^ (unsigned long long)__double_as_longlong(b.r)) |
         ((unsigned long long)__double_as_longlong(a.ma) ^ (unsigned long long)__double_as_longlong(b.ma)) |
         ((unsigned long long)__double_as_longlong(a.mb) ^ (unsigned long long)__double_as_longlong(b.mb)) |
         ((unsigned long long)__double_as_longlong(a.e) ^ (unsigned long long)__double_as_longlong(b.e));
}

// Column-phase source for walk_strip: the U_a ring (4-row chunks, kFNBA
// buffers, one full barrier each) read through a cursor, the U_b slot rows
// written through another, and the hand-over (Chunk callback) at every
// completed 4-row output chunk.  kTight: walk_strip runs steady uniform runs
// through peek/preload (the cells are consumed in order either way).
template <class Chunk>
struct FusedCol {
  static constexpr bool kTight = true;
  Chunk& chunk;
  uint32_t ring;      // hb_smem offset of ring buffer 0 + this lane's column
  uint32_t bars;      // hb_smem offset of the kFNBA full barriers
  int ka;             // first output strip cell
  bool active;
  // load cursor: next cell's address, cells left in its chunk, its chunk number
  uint32_t lo_at;
  int lo_left;
  unsigned lo_q;
  uint32_t at1, at2, at3;  // addresses of the last three cells taken (at3: the cell updated next)
  Cons last, before;       // the last two cells taken (the uniform-window test)
  Cons pre;                // a cell peeked by the tight loop, not yet taken
  bool have;
  // output cursor: the slot row address of the next updated cell (this
  // lane's column), outputs left in the chunk / after it
  uint32_t out_at, lane_off;
  int out_left, out_rest, q;
  unsigned nskip;
  int skip_cool;
  uint32_t memo_at;
  bool memo_valid;
  bool cross;  // steady uniform run: every active lane of the warp holds the same state
  bool counted;  // an output strip of the band (the halo strips' updates are not counted)

  // column orientation: mom_a = mom_x (var 1), mom_b = mom_y (var 2)
  __device__ __forceinline__ static Cons get(uint32_t at) {
    const uint8_t* b = hb_smem + at;
    return {*(const double*)b, *(const double*)(b + kFVarBytesA),
            *(const double*)(b + 2 * kFVarBytesA), *(const double*)(b + 3 * kFVarBytesA)};
  }
  __device__ __forceinline__ void wait_chunk() const {
    mbar_wait((uint64_t*)(hb_smem + bars) + (lo_q & (kFNBA - 1)), (lo_q / kFNBA) & 1u);
  }
  // item start: the first cell taken is input row i_a - 2 (row 2 of chunk 0)
  __device__ __forceinline__ void begin(unsigned q0) {
    lo_q = q0;
    lo_at = ring + (q0 & (kFNBA - 1)) * kFChunkBytes + 2 * kFRowBytesA;
    lo_left = 2;
    have = false;
    wait_chunk();
  }
  __device__ __forceinline__ Cons peek(int) {
    if (lo_left == 0) {
      ++lo_q;
      lo_at = ring + (lo_q & (kFNBA - 1)) * kFChunkBytes;
      lo_left = 4;
      wait_chunk();
    }
    at3 = at2;
    at2 = at1;
    at1 = lo_at;
    lo_at += kFRowBytesA;
    --lo_left;
    return get(at1);
  }
  __device__ __forceinline__ void preload(const Cons& u) {
    pre = u;
    have = true;
  }
  __device__ __forceinline__ Cons load(int k) {
    const Cons u = have ? pre : peek(k);
    have = false;
    before = last;
    last = u;
    return u;
  }
  // ---- whole chunks of a steady uniform run (walk_strip's tight loop) ----------
  __device__ __forceinline__ void enter_tight(const Cons& u) {
    cross = __all_sync(0xffffffffu, same_bits(u, shfl(u, 0)) || !active);
  }
  // the cursors sit on a chunk boundary: four outputs open a slot, their four
  // incoming cells are rows 2-3 of this input chunk and rows 0-1 of the next
  __device__ __forceinline__ bool chunk_aligned() const {
    return out_left == 4 && lo_left == 2 && !have;
  }
  __device__ __forceinline__ bool chunk_equal(const Cons& u) const {
    const unsigned nq = lo_q + 1;
    const uint32_t nx_at = ring + (nq & (kFNBA - 1)) * kFChunkBytes;
    mbar_wait((uint64_t*)(hb_smem + bars) + (nq & (kFNBA - 1)), (nq / kFNBA) & 1u);
    const unsigned long long d = diff_bits(get(lo_at), u) | diff_bits(get(lo_at + kFRowBytesA), u) |
                                 diff_bits(get(nx_at), u) | diff_bits(get(nx_at + kFRowBytesA), u);
    return d == 0ull;
  }
  // takes those four cells (all equal to o.un) and hands the chunk over
  template <class Sink>
  __device__ __forceinline__ void take_chunk(Sink& sink, int c, const StepOut& o) {
    ++lo_q;
    const uint32_t nx_at = ring + (lo_q & (kFNBA - 1)) * kFChunkBytes;
    at3 = lo_at + kFRowBytesA;
    at2 = nx_at;
    at1 = nx_at + kFRowBytesA;
    lo_at = nx_at + 2 * kFRowBytesA;
    // lo_left stays 2; last/before already hold this state
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      sink(c + k, o);
      out_at += kFRowBytesS;
    }
    if (counted) nskip += 4;
    const bool last_chunk = out_rest == 0;
    out_at = chunk(q++, last_chunk, cross, o.un) + lane_off;
    out_left = out_rest < 4 ? out_rest : 4;
    out_rest -= out_left;
  }
  __device__ __forceinline__ Cons reload(int) const { return get(at3); }
  __device__ __forceinline__ Cons prev() const { return before; }
  __device__ __forceinline__ void count_skip() { nskip += counted ? 1u : 0u; }
  // after iteration c: cell c-1 was updated (c > ka); a completed 4-row
  // output chunk (or the item's last) is handed over
  __device__ __forceinline__ void boundary(int c) {
    if (c > ka) {
      out_at += kFRowBytesS;
      if (--out_left == 0) {
        const bool last_chunk = out_rest == 0;
        out_at = chunk(q++, last_chunk, false, Cons{}) + lane_off;
        out_left = out_rest < 4 ? out_rest : 4;
        out_rest -= out_left;
      }
    }
  }
};

template <int LAST, bool PEER, int FLUX>
__global__ void __launch_bounds__(256, 1)
    sweep_xy_kernel(SweepArgs a, const __grid_constant__ CUtensorMap load_map,
                    const __grid_constant__ CUtensorMap store_map) {
  pdl_launch_dependents();
  const uint32_t pad = (128u - (smem_u32(hb_smem) & 127u)) & 127u;
  const uint32_t ring0 = pad, slots0 = pad + kFSlotOff, bars = pad + kFBarOff;
  FusedHdr* const hdrs = (FusedHdr*)(hb_smem + pad + kFHdrOff);
  int* const flags = (int*)(hb_smem + pad + kFFlagOff);  // [0] claimed item, [1] redo vote
  FusedUni* const unis = (FusedUni*)(hb_smem + pad + kFUniOff);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int q = 0; q < kFNBA; ++q) mbar_init((uint64_t*)(hb_smem + bars) + q, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const Gas g = make_gas(a.gamma);
  pdl_wait();
  if (latched(a)) return;
  if (*(volatile unsigned long long*)a.dt_err != kNoError) {
    if (blockIdx.x == 0 && tid == 0) record(a.err, *(volatile unsigned long long*)a.dt_err);
    return;
  }
  const double dt = step_dt(a);
  const int nx = a.nx, ny = a.ny;
  const bool refl = a.bc == 0;
  unsigned nskip = 0;      // uniform-window updates of this thread's role
  double spd_max = 0.0;    // row warps: dt signal speeds
  unsigned long long dt_key = kNoError;

  if (warp < 4) {
    // ---- column phase (warps 0-3, one lane per strip) -------------------------
    const double dtdx = dt / a.dx;  // euler_kernel.cpp:112 along the column axis
    const int nbands = (ny + kFW - 1) / kFW;
    const int items = nbands * a.nseg;
    unsigned q0 = 0;   // running input-chunk number (ring bookkeeping)
    unsigned m = 0;    // running published-chunk number (slots)
    int seq = 0;       // items taken by this CTA
    int skip_cool = 0;
    bool memo_keep = false;  // exact-10: this thread's interface memo holds an exact entry
    auto acquire = [&](unsigned mm) {  // slot of chunk mm free (its chunk mm-3 was taken)
      if (mm >= kFNS) bar_sync(kFBarEmpty + (int)(mm % kFNS), 256);
    };
    for (;; ++seq) {
      if (tid == 0) {
        flags[0] = (int)atomicAdd(a.counter, 1u);
        flags[1] = 0;
      }
      bar_sync(kFBarCol, 128);
      const int item = flags[0];
      if (item >= items) break;
      const int band = item % nbands, sg = item / nbands;
      const int j0 = band * kFW + 1;
      const int i_a = 1 + sg * a.seg;
      const int i_b = min(nx, i_a + a.seg - 1);
      const int ka = i_a + 1, kb = i_b + 1;
      const int nq = (i_b + 2 - (i_a - 4)) / 4 + 1;  // input chunks: rows i_a-4 .. i_b+2
      const int tj_load = (j0 - 8 + kColOff) >> 3;   // block of column j0-8
      const int s = tid;                             // strip -> column j0-2+s
      const int j = j0 - 2 + s;
      const bool active = s < kFStrips && j >= 1 && j <= ny;
      const bool edge = active && (j <= 2 || j >= ny - 1);
      // a band whose 124 strips are all interior columns (no wall ghosts, no
      // inactive strips): its uniform chunks are uniform rows
      const bool plain = j0 - 2 > 2 && j0 + kFW + 1 < ny - 1;
      const unsigned long long base_x = error_key(a.step, 1, j, 0, 0, 0);
      auto issue = [&](int q) {  // tid 0: input chunk q of this item
        const int rr = i_a - 4 + 4 * q - 1;  // grid row - 1 of its first row
        const unsigned n = q0 + (unsigned)q;
        uint64_t* bar = (uint64_t*)(hb_smem + bars) + (n % kFNBA);
        mbar_expect_tx(bar, kFChunkBytes);
        tma_load5(hb_smem + ring0 + (n % kFNBA) * kFChunkBytes, &load_map, bar, 0, tj_load, rr & 31,
                  0, (rr >> 5) + 1);
      };
      unsigned long long ek = kNoError;
      auto pass = [&](auto math, int pass_no) {
        using M = decltype(math);
        bar_sync(kFBarCol, 128);  // the ring is free
        if (tid == 0)
          for (int q = 0; q < kFNBA && q < nq; ++q) issue(q);
        acquire(m);
        // publishes chunk q (slot m % kFNS); returns the slot row base of the next
        auto chunk = [&](int q, bool last, bool uni, const Cons& st) -> uint32_t {
          const unsigned sl = m % kFNS;
          if (lane == 0) {
            FusedUni& fu = unis[sl];
            fu.uni[warp] = uni && plain;
            if (uni) {
              fu.st[warp][0] = st.r;
              fu.st[warp][1] = st.ma;
              fu.st[warp][2] = st.mb;
              fu.st[warp][3] = st.e;
            }
          }
          if (tid == 0) {
            FusedHdr& h = hdrs[sl];
            h.tag = 2 * seq + pass_no;
            h.i0 = i_a + 4 * q;
            h.nrows = min(4, i_b - h.i0 + 1);
            h.j0 = j0;
            h.first = q == 0;
            h.end = 0;
          }
          fence_async_smem();  // slot writes -> the row warps' TMA stores (skipped rows)
          bar_arrive(kFBarFull + (int)sl, 256);
          ++m;
          // input chunk q is free once every column warp is here: the next
          // slot's barrier (all 128 column threads sync on it) says so, else
          // the column warps' own
#if HB_FONEBAR
          const bool joined = !last && m >= (unsigned)kFNS;
          if (joined) acquire(m);
          else bar_sync(kFBarCol, 128);
#else
          const bool joined = false;
          bar_sync(kFBarCol, 128);
#endif
          if (tid == 0 && q + kFNBA < nq) {
            fence_async_smem();
            issue(q + kFNBA);
          }
          if (!last && !joined) acquire(m);
          return slots0 + (m % kFNS) * kFSlotBytes;
        };
        FusedCol<decltype(chunk)> col{chunk};
        col.ring = ring0 + (uint32_t)(s + 6) * 8;
        col.bars = bars;
        col.ka = ka;
        col.active = active;
        col.counted = active && s >= 2 && s < kFW + 2;
        col.begin(q0);
        col.lane_off = (uint32_t)(s + 14) * 8;
        col.out_at = slots0 + (m % kFNS) * kFSlotBytes + col.lane_off;
        col.out_left = min(4, kb - ka + 1);
        col.out_rest = kb - ka + 1 - col.out_left;
        col.q = 0;
        col.nskip = 0;
        col.skip_cool = skip_cool;
        col.memo_at = pad + kFMemoOff + (uint32_t)tid * 8;  // exact-10 interface memo (13 x 1 KB)
        col.memo_valid = memo_keep;  // kept across this thread's work items while exact
        auto put_slot = [&](uint32_t at, const Cons& u) {
          double* q = (double*)(hb_smem + at);
          q[0] = u.r;
          q[kFPos] = u.ma;
          q[2 * kFPos] = u.mb;
          q[3 * kFPos] = u.e;
        };
        auto sink = [&](int, const StepOut& o) {
          if (active) put_slot(col.out_at, o.un);
          if (edge) {  // y-wall ghosts of the column-sweep output (grid.cpp:44-59)
            const uint32_t row = col.out_at - col.lane_off;
            auto ghost = [&](int jt, bool neg) {
              Cons gh = o.un;
              if (neg) gh.mb = -gh.mb;
              put_slot(row + (uint32_t)(jt - j0 + 16) * 8, gh);
            };
            if (refl) {
              if (j <= 2) ghost(1 - j, true);
              if (j >= ny - 1) ghost(2 * ny + 1 - j, true);
            } else {
              if (j == 1) { ghost(0, false); ghost(-1, false); }
              if (j == ny) { ghost(ny + 1, false); ghost(ny + 2, false); }
            }
          }
        };
        ek = kNoError;
        const bool ok = walk_strip<M, false, FLUX>(ka, kb, col, sink, g, dtdx, 0.0, base_x, a.row0, ek);
        q0 += (unsigned)nq;
        memo_keep = col.memo_valid;
        skip_cool = col.skip_cool;
        nskip += col.nskip;
        return ok || !active;
      };
      if (!pass(FastMath{}, 0)) flags[1] = 1;
      bar_sync(kFBarCol, 128);
      if (flags[1]) pass(ExactMath{}, 1);  // a fast pass left its proven range: redo the item
      if (active && ek != kNoError) record(a.err, ek);
    }
    // end of the chunk stream, then the row warps' last slot releases
    acquire(m);
    if (tid == 0) {
      hdrs[m % kFNS].end = 1;
      hdrs[m % kFNS].first = 0;
    }
    bar_arrive(kFBarFull + (int)(m % kFNS), 256);
    for (int k = 1; k < kFNS; ++k) acquire(m + k);
  } else {
    // ---- row phase (warps 4-7: row w-4 of each chunk, lane-parallel) ----------
    const double dtdx = dt / a.dx2;
    const int wr = warp - 4;
    double* __restrict__ dst = a.dst;
    const size_t pitch = a.pitch;
    RowMemo memo{};
    memo.valid = false;
    EdgeMemo* const edge = (EdgeMemo*)(hb_smem + pad + kFEdgeOff) + 2 * wr;
    if (lane < 2) edge[lane].valid = 0.0;
    __syncwarp();
    bool wrote_peer = false;
    RowAcc acc, done;
    acc.clear();
    done.clear();
    int cur = -1;          // tag of the pass being accumulated
    bool redo_wait = false;
    for (unsigned n = 0;; ++n) {
      const unsigned sl = n % kFNS;
      bar_sync(kFBarFull + (int)sl, 256);
      if (n >= (unsigned)kFLag) {  // the stores of chunk n - kFLag have read their slot: release it
        if (lane == 0) {
          if constexpr (kFLag == 1) bulk_wait_read0();
          else bulk_wait_read1();
        }
        __syncwarp();
        bar_arrive(kFBarEmpty + (int)((n - kFLag) % kFNS), 256);
      }
      const FusedHdr h = hdrs[sl];
      if (h.end) {  // the slots still held
        if (lane == 0) bulk_wait_read0();
        __syncwarp();
        for (unsigned r = n >= (unsigned)kFLag ? n - kFLag + 1 : 0; r < n; ++r)
          bar_arrive(kFBarEmpty + (int)(r % kFNS), 256);
        break;
      }
      if (h.first) {
        // a redo pass of the same item supersedes the fast pass's
        // contributions; otherwise the previous pass is final
        if (cur >= 0 && (cur >> 1) != (h.tag >> 1)) done.add(acc);
        redo_wait = cur >= 0 && (cur >> 1) == (h.tag >> 1);
        acc.clear();
        cur = h.tag;
      }
      if (wr >= h.nrows) {  // no row for this warp: an empty group keeps one group per chunk
        if (lane == 0) bulk_commit();
        continue;
      }
      const int i = h.i0 + wr;
      const int gi = a.row0 + i;
      const uint32_t at = slots0 + sl * kFSlotBytes + wr * kFRowBytesS;
      const bool lo = a.wall_lo && i <= 2, hi = a.wall_hi && i >= nx - 1;
      // slab borders: the rows the neighbours' next column sweep needs go into
      // their inboxes over NVLink (InterfaceBuffer, decomposition.hpp:58-79)
      const bool up = PEER && a.halo_up && i <= 2, dn = PEER && a.halo_dn && i >= nx - 1;
      // a chunk every column warp published as uniform, all in one state this
      // warp has already evaluated to the identity in this launch: the row
      // keeps its input (fused_row would find exactly this by reading it)
      bool quick = false;
      if (memo.valid && !(lo || hi || up || dn)) {
        const FusedUni& fu = unis[sl];
        const int4 uf = *(const int4*)fu.uni;
        if (uf.x & uf.y & uf.z & uf.w) {
          // row orientation: mom_a = mom_y (st[2]), mom_b = mom_x (st[1])
          unsigned long long d = 0ull;
#pragma unroll
          for (int w2 = 0; w2 < 4; ++w2) {
            const double2 ab = *(const double2*)&fu.st[w2][0], cd = *(const double2*)&fu.st[w2][2];
            d |= diff_bits(Cons{ab.x, cd.x, ab.y, cd.y}, memo.u);
          }
          quick = d == 0ull;
        }
      }
      if (quick) {
        if (lane >= 1 && lane <= 30) acc.nskip += 4;
        acc.spd = smax(acc.spd, memo.spd);
      } else {
      RowGeo rg;
      rg.j0 = h.j0;
      rg.jb = h.j0 - 4 + 4 * lane;
      rg.jlo = h.j0 - 2 > -1 ? h.j0 - 2 : -1;
      rg.jhi = h.j0 + kFW + 1 < ny + 2 ? h.j0 + kFW + 1 : ny + 2;
      rg.ohi = h.j0 + kFW - 1 < ny ? h.j0 + kFW - 1 : ny;
      rg.key_base = error_key(a.step, 2, gi, 0, 0, 0);
      rg.dt_base = error_key(a.step + 1, 0, gi, 0, 0, 0);
      Cons uin[4], out[4];
      bool outk[4];
      fused_row<FLUX>(at, lane, rg, ny, g, dtdx, memo, edge, acc, uin, out, outk);
      // x-wall ghost rows (grid.cpp:26-42): of the next step, from this row's
      // update -- or, in the run's last step, the ones the reference leaves
      // behind: its last apply_boundary ran on the column-sweep output
      // (schedulers.cpp:103-116), this row's input
      if (lo || hi) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (!outk[k]) continue;
          const int jj = rg.jb + k;
          Cons gh = LAST ? uin[k] : out[k];
          auto put = [&](int ii) {
            double* q2 = dst + cell_index(pitch, 0, ii, jj);
            q2[0] = gh.r;
            q2[kVarStep] = gh.mb;
            q2[2 * kVarStep] = gh.ma;
            q2[3 * kVarStep] = gh.e;
          };
          if (refl) {
            gh.mb = -gh.mb;  // row orientation: mom_b is mom_x
            put(lo ? 1 - i : 2 * nx + 1 - i);
          } else if (lo && i == 1) {
            put(0);
            put(-1);
          } else if (hi && i == nx) {
            put(nx + 1);
            put(nx + 2);
          }
        }
      }
      if constexpr (PEER) {
        if (up || dn) {
          auto put_peer = [&](double* q, const Cons& u) {  // row orientation: mom_b is mom_x
            q[0] = u.r;
            q[2 * pitch] = u.ma;
            q[pitch] = u.mb;
            q[3 * pitch] = u.e;
          };
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            if (!outk[k]) continue;
            const int jj = rg.jb + k;
            if (up) put_peer(a.halo_up + (size_t)(i - 1) * 4 * pitch + (jj + kColOff), out[k]);
            if (dn) put_peer(a.halo_dn + (size_t)(i - (nx - 1)) * 4 * pitch + (jj + kColOff), out[k]);
          }
          wrote_peer = true;
        }
      }
      }  // !quick
      if (LAST && (h.j0 == 1 || h.j0 + kFW - 1 >= ny) && lane < 16) {
        // the run's final y-wall ghost columns: the column-sweep output's
        // (grid.cpp:44-59), which the row phase left in the slot untouched
        const int v = lane & 3, cg = lane >> 2;            // cg 0, 1: columns -1, 0; 2, 3: ny+1, ny+2
        const int jg = cg < 2 ? cg - 1 : ny - 1 + cg;
        if (cg < 2 ? h.j0 == 1 : h.j0 + kFW - 1 >= ny)
          dst[cell_index(pitch, v, i, jg)] =
              *(const double*)(hb_smem + at + v * kFVarBytesS + (uint32_t)(jg - h.j0 + 16) * 8);
      }
      fence_async_smem();
      __syncwarp();
      if (lane == 0) {
        if (redo_wait) bulk_wait0();  // the superseded pass's stores of these rows have landed
        const int rr = i - 1;
        const int tj_store = (h.j0 + kColOff) >> 3;
        for (int v = 0; v < 4; ++v)
          tma_store5(&store_map, hb_smem + at + v * kFVarBytesS + 16 * 8, 0, tj_store, rr & 31, v,
                     (rr >> 5) + 1);
        bulk_commit();
      }
      redo_wait = false;
    }
    if (cur >= 0) done.add(acc);
    // peer stores performed system-wide before this kernel completes (the
    // neighbour reads them after the dt exchange that follows on the stream)
    if (PEER && wrote_peer) __threadfence_system();
    if (done.ekey != kNoError) record(a.err, done.ekey);
    spd_max = done.spd;
    dt_key = done.dtkey;
    nskip = done.nskip;
  }
  if (lane == 0) bulk_wait0();
  {
    unsigned n = nskip;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
    if (lane == 0 && a.skipped && n) atomicAdd(a.skipped + (warp < 4 ? 0 : 1), (unsigned long long)n);
  }
  if (a.want_limit && warp >= 4) {
    const double smx = __longlong_as_double(
        (long long)~warp_min_u64(~(unsigned long long)__double_as_longlong(spd_max)));
    const unsigned long long e = warp_min_u64(dt_key);
    if (lane == 0) {
      if (smx > 0.0) atomicMin(a.limit_out, (unsigned long long)__double_as_longlong(a.spacing / smx));
      if (e != kNoError) atomicMin(a.dt_err, e);
    }
  }
  // the last CTA to finish resets this step's dt slot (the step after next
  // writes it) and the work counter
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    const unsigned prev = atomicAdd(a.done, 1u);
    if (prev == gridDim.x - 1) {
      if (!LAST) *a.limit_in = kEmptyLimit;  // (a run's last dt stays readable)
      *a.counter = 0u;
      *a.done = 0u;
      __threadfence();
    }
  }
}
