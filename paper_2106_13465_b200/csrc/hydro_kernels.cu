// hydro_kernels.cu -- the fused sweep kernels of the HYDRO step (sm_100a).
//
// One step of the reference (proj/src/schedulers.cpp:103-116) is
//   apply_boundary -> compute_dt -> column sweep -> apply_boundary -> row sweep.
// Split schedule: two launches per step --
//   sweep_x  (Column axis, strips along i): reads U_a, writes U_b, and writes
//            the j-ghost columns of U_b (the y-wall half of the second
//            apply_boundary, grid.cpp:44-59) from its own outputs;
//   sweep_y  (Row axis, strips along j): reads U_b, writes U_a, writes the
//            i-ghost rows of U_a for the next step (the x-wall half of
//            apply_boundary, grid.cpp:26-42), and folds cell_dt_limit of the
//            new state into the next step's dt (compute_dt, :233-242).
// Fused schedule: one launch per step (sweep_xy_kernel, hydro_fused.cuh,
// included below): the same two phases with U_b kept in shared memory.
// Every thread owns one strip segment and walks it with a register sliding
// window: primitive conversion, minmod slopes, Hancock predictor, evolved
// faces, HLLC flux and the conservative update of the reference's four strip
// loops (euler_kernel.cpp:111-223) are fused; no per-strip scratch touches
// HBM.  Segments overlap by the 2-cell stencil halo only.
//
// Memory paths: the state is tiled in HBM (32 rows x 8 columns x 4 variables
// per 8 KB block, cell_index in hydro_kernels.cuh); both sweeps stage their
// strips through per-warp rings in shared memory, filled and drained by TMA
// (cp.async.bulk.tensor.5d over the tiled view, mbarrier completion) and used
// in place (Tiles below).  The column sweep's warp holds 32 adjacent columns:
// each chunk is one box of 4 grid rows x 4 variables x 4 column blocks
// (sixteen 256-byte pieces).  The row sweep's warp holds 32 adjacent rows:
// each chunk is one box of 32 rows x 8 (bitwise HLLC, SWIZZLE_64B) or 4
// (tolerance HLLC and exact-10, SWIZZLE_32B) columns x 4 variables, i.e. a
// contiguous piece of a block and a transposed tile from the walker's point
// of view.  Warps claim work items (32 strips x one segment) dynamically from
// a per-sweep counter, in bands of strip groups (item_coords), and redo an
// item with the exact math policy if the fast pass left its proven range.
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "hydro_exact.cuh"
#include "hydro_kernels.cuh"

// The same sweeps are compiled a second time by hydro_kernels_tol.cu with
// HB_TOLERANCE (tolerance math mode): only the sweep kernels
// and their launchers, exported with a _tol suffix.
#ifdef HB_TOLERANCE
#define HB_SWEEP(name) name##_tol
#else
#define HB_SWEEP(name) name
#endif

namespace hb {

namespace {

constexpr unsigned long long kEmptyLimit = ~0ull;  // sentinel above every positive double

__device__ __forceinline__ unsigned long long warp_min_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
    v = (w < v) ? w : v;
  }
  return v;
}

// ---------------------------------------------------------------------------
// The strip walker.

// Carried from one cell to the next.  The conserved cells themselves are
// not carried: the update re-reads cell c-1 from L1 / shared memory, which
// costs 4 loads instead of 16 register moves and 16 live registers per cell.
struct Window {
  Prim wA, wB;      // primitives of cells c-1, c
  Face frPrev;      // right face of cell c-1
  Flux fluxPrev;    // flux through interface c-2 | c-1
};

struct StepOut {
  Prim wC;          // primitive of the incoming cell c+1
  int fC;           // its positivity failure (-1 none)
  Face fl, fr;      // faces of cell c
  Flux F;           // flux through interface c-1 | c
  int fR;           // Riemann failure (exact-10: 3 = vacuum), -1 none
  Cons un;          // cell c-1 after the conservative update
  int fU;
  double spd;       // dt signal speed of the updated cell (row sweep)
  int fD;
};

// One walker iteration at cell c.  STAGE 0: primitive + faces only (the
// first halo iteration); STAGE 1: + flux (second halo iteration);
// STAGE 2: + conservative update (+ dt limit).
// FLUX 0: HLLC (euler_kernel.cpp:59-109); FLUX 1: exact Riemann, 10 Newton
// iterations (hydro_exact.cuh).
extern __shared__ __align__(128) uint8_t hb_smem[];

// Exact-10 interface memo (per thread, in shared memory after the tiles):
// the last Riemann problem this walk solved -- both face states bit for bit
// -- and its flux.  The solver is a pure function of the two states, so an
// interface whose states repeat the previous one's (uniform flow, where the
// exact solver is as expensive as anywhere) takes the stored flux: the same
// bits without the Newton/log/exp work.  An entry is reused only while it
// is exact: within a pass (whose range tests it is folded into), and across
// the thread's work items only after an exact pass or a fast pass that kept
// every range (walk_strip's memo_valid hand-over).
struct Memo {
  uint32_t at;  // hb_smem offset of this thread's field 0 (fields 1 KB apart)
  bool valid;
  __device__ __forceinline__ double& f(int k) const {
    return *(double*)(hb_smem + at + k * 1024);
  }
  __device__ __forceinline__ static bool same(double a, double b) {
    return __double_as_longlong(a) == __double_as_longlong(b);
  }
  __device__ __forceinline__ bool match(const Prim& a, const Prim& b) const {
    return valid & same(f(0), a.r) & same(f(1), a.va) & same(f(2), a.vb) & same(f(3), a.p) &
           same(f(4), b.r) & same(f(5), b.va) & same(f(6), b.vb) & same(f(7), b.p);
  }
  __device__ __forceinline__ void put(const Prim& a, const Prim& b, const Flux& F, bool vac) {
    f(0) = a.r; f(1) = a.va; f(2) = a.vb; f(3) = a.p;
    f(4) = b.r; f(5) = b.va; f(6) = b.vb; f(7) = b.p;
    f(8) = F.m; f(9) = F.ma; f(10) = F.mb; f(11) = F.e;
    f(12) = vac ? 1.0 : 0.0;
    valid = true;
  }
};
struct NoMemo {
  bool valid;
};

template <int FLUX, class M, class Mem>
__device__ __forceinline__ Flux riemann(M& m, const Face& L, const Face& R, const Gas& g, int& fail,
                                        Mem& memo) {
  fail = -1;
  if constexpr (FLUX == 0) {
    return hllc(m, L, R, g);
  } else {
    bool vacuum;
    Flux f;
    if constexpr (std::is_same_v<Mem, NoMemo>) {  // (the fused step's row phase)
      f = exact10_flux(m, L, R, g, vacuum);
    } else if (memo.match(L.w, R.w)) {
      f = {memo.f(8), memo.f(9), memo.f(10), memo.f(11)};
      vacuum = memo.f(12) != 0.0;
    } else {
      f = exact10_flux(m, L, R, g, vacuum);
      memo.put(L.w, R.w, f, vacuum);
    }
    if (vacuum) {
      if constexpr (M::kFast) m.fallback();  // reported by the exact pass
      else fail = 3;
    }
    return f;
  }
}

#ifndef HB_FOLD_EXACT
#define HB_FOLD_EXACT 1
#endif
#ifndef HB_FOLD_HLLC
#define HB_FOLD_HLLC 0
#endif

template <int STAGE, bool WANT_DT, int FLUX, class M, class Old, class Mem>
__device__ __forceinline__ void step_cell(M& m, const Window& w, const Cons& uC, double half,
                                          double dtdx, double spacing, const Gas& g,
                                          const Old& old, StepOut& o, Mem& memo,
                                          bool upd = true) {
  o.fC = to_prim(m, uC, g, o.wC);
  Cons el, er;
  predict_evolved(m, w.wA, w.wB, o.wC, half, g, el, er);
  // left face first: it meets the previous right face in this iteration's
  // Riemann problem, after which that face is dead and the new right face
  // can take its registers
  // (the first halo iteration's left face would only meet the interface
  // before the segment's halo: it is not evaluated)
  if (STAGE >= 1) o.fl = face_prim(m, el, w.wB, g);
  o.fR = -1;
  if (STAGE >= 1) o.F = riemann<FLUX>(m, w.frPrev, o.fl, g, o.fR, memo);
  o.fr = face_prim(m, er, w.wB, g);
  if (STAGE >= 2 && upd) {
    o.un = old();
#ifdef HB_TOLERANCE
    if constexpr (!WANT_DT) {
      o.fU = update_cell_nodt(m, o.un, w.fluxPrev, o.F, dtdx);
    } else
#endif
    {
      Recip rn;
      UpdAux aux;
      o.fU = update_cell(m, o.un, w.fluxPrev, o.F, dtdx, rn, aux);
      if (WANT_DT) o.fD = dt_speed(m, o.un, rn, aux, g, o.spd);
    }
  }
}

__device__ __forceinline__ void record(unsigned long long* err, unsigned long long key) {
  atomicMin(err, key);
}

struct OkKey {
  bool ok;
  unsigned long long key;
};
__device__ __forceinline__ OkKey make_pair_ok(bool ok, unsigned long long key) { return {ok, key}; }

__device__ __forceinline__ void keep_min(unsigned long long& k, unsigned long long v) {
  k = v < k ? v : k;
}

// Walks strip cells [ka, kb] (strip coordinates: cell k holds grid index
// k-1) with math policy M.  src.load(k) returns cell k in sweep orientation
// (called for k = ka-2 .. kb+2 in order), sink(k, out) receives updated
// cells ka..kb, src.boundary(c) is called after every iteration (chunk
// bookkeeping).  Positivity failures are folded into `ekey` (kg converts a
// local strip cell to the global index used in error keys).  The two halo
// iterations are peeled, so a segment costs its cells plus two primitive
// conversions, two face reconstructions and one flux.  Returns false if a
// FastMath operation left its proven range somewhere in the segment.
// Main-loop unroll: 2 for the tolerance row sweep (its 168-register budget
// holds the renamed window: -2..6% on configs 1-2), 1 elsewhere (the column
// sweeps spill at their 128-register cap, the bitwise row sweep runs slower).
#ifndef HB_UNROLL
#ifdef HB_TOLERANCE
#define HB_UNROLL 2
#else
#define HB_UNROLL 1
#endif
#endif

__device__ __forceinline__ bool same_bits(const Cons& a, const Cons& b) {
  return (__double_as_longlong(a.r) == __double_as_longlong(b.r)) &
         (__double_as_longlong(a.ma) == __double_as_longlong(b.ma)) &
         (__double_as_longlong(a.mb) == __double_as_longlong(b.mb)) &
         (__double_as_longlong(a.e) == __double_as_longlong(b.e));
}

// The uniform-window identity (below) pays where the sweeps are compute-bound
// on uniform flow: bitwise config 3 column/row sweeps -11%/-22%, config 1
// -20%/-36%; tolerance config 3 -11%/-10%, config 1 -10%/-13%.  Dense flow
// runs a walker without it (walk_strip).
#ifndef HB_SKIP
#define HB_SKIP 1
#endif

// Walks strip cells [ka, kb] (strip coordinates: cell k holds grid index
// k-1) with math policy M.  src.load(k) returns cell k in sweep orientation
// (called for k = ka-2 .. kb+2 in order), sink(k, out) receives updated
// cells ka..kb, src.boundary(c) is called after every iteration (chunk
// bookkeeping).  Positivity failures are folded into `ekey` (kg converts a
// local strip cell to the global index used in error keys).  The two halo
// iterations are peeled, so a segment costs its cells plus two primitive
// conversions, two face reconstructions and one flux.  Returns false if a
// FastMath operation left its proven range somewhere in the segment.
//
// Uniform-window identity: the update of cell c-1 is a pure function of the
// five cells c-3..c+1 (loop 1-4 of sweep_strip, euler_kernel.cpp:111-223),
// and so are the carried faces and flux.  When the six cells c-4..c+1 are
// bitwise equal, cell c-1's window equals cell c-2's, so its update is cell
// c-2's result bit for bit, and the carried window state is unchanged; if
// that result was the identity (the updated cell equal to its input), cell
// c-1 keeps its input and nothing needs evaluating -- the same bits as
// evaluating it (uniform flow, e.g. the quiescent gas ahead of a blast).  A
// warp takes the shortcut only when all its lanes can (no divergence), in
// either math policy; errors are reported by the first cell of a uniform run,
// which is evaluated (later ones would fail identically at higher indices).
template <class M, bool WANT_DT, int FLUX, bool SKIP, class Src, class Sink>
__device__ __forceinline__ bool walk_strip_impl(int ka, int kb, Src& src, Sink& sink, const Gas& g,
                                                double dtdx, double spacing,
                                                unsigned long long key_base, int kg,
                                                unsigned long long& ekey) {
  M m;
  if constexpr (M::kFast) m.ok = g.fast;  // divb's bounds need gamma - 1 in [2^-6, 2^6]
  const double half = 0.5 * dtdx;
  using Mem = std::conditional_t<FLUX == 1, Memo, NoMemo>;
  Mem memo{};
  if constexpr (FLUX == 1) memo.at = src.memo_at;
  memo.valid = src.memo_valid;
  Window w;
  auto none = [] { return Cons{}; };
  int same = 0;         // consecutive loaded cells bitwise equal to their predecessor
  bool idprev = false;  // the last update was the identity
  // A warp whose last item had no uniform window at all (dense flow) stops
  // testing for kSkipCool items: the cell compares cost ~5% where they never
  // pay off.
  constexpr int kSkipCool = 8;
  constexpr bool kSkip = SKIP;
  const bool probe = kSkip && src.skip_cool == 0;
  bool saw = false;
  Cons u = src.load(ka - 2);
  int f = to_prim(m, u, g, w.wA);
  if (f >= 0) keep_min(ekey, key_base | ((unsigned long long)(ka - 2 + kg) << 2) | f);
  {
    const Cons u1 = src.load(ka - 1);
    if (probe) same = same_bits(u1, u) ? 1 : 0;
    u = u1;
  }
  f = to_prim(m, u, g, w.wB);
  if (f >= 0) keep_min(ekey, key_base | ((unsigned long long)(ka - 1 + kg) << 2) | f);
  {  // c = ka-1: faces of the first halo cell
    const Cons uC = src.load(ka);
    if (probe) same = same_bits(uC, u) ? same + 1 : 0;
    StepOut o;
    step_cell<0, false, FLUX>(m, w, uC, half, dtdx, spacing, g, none, o, memo);
    if (o.fC >= 0) keep_min(ekey, key_base | ((unsigned long long)(ka + kg) << 2) | o.fC);
    src.boundary(ka - 1);
    w.wA = w.wB;
    w.wB = o.wC;
    w.frPrev = o.fr;
  }
  // FOLD: the c = ka iteration runs in the main loop with its update
  // skipped, so the walker holds one copy of the Riemann solve (the exact-10
  // solver is ~5k instructions per copy: instruction-cache pressure)
  constexpr bool kFold = FLUX == 1 ? HB_FOLD_EXACT : HB_FOLD_HLLC;
  if constexpr (!kFold) {  // c = ka: faces of cell ka and the flux through its left interface
    const Cons uC = src.load(ka + 1);
    if (probe) same = same_bits(uC, src.prev()) ? same + 1 : 0;
    StepOut o;
    step_cell<1, false, FLUX>(m, w, uC, half, dtdx, spacing, g, none, o, memo);
    if (o.fC >= 0) keep_min(ekey, key_base | ((unsigned long long)(ka + 1 + kg) << 2) | o.fC);
    if (o.fR >= 0)
      keep_min(ekey, key_base | (1ull << 20) | ((unsigned long long)(ka - 1 + kg) << 2) | o.fR);
    src.boundary(ka);
    w.wA = w.wB;
    w.wB = o.wC;
    w.frPrev = o.fr;
    w.fluxPrev = o.F;
  }
  constexpr int kUnroll = (WANT_DT && FLUX == 0) ? HB_UNROLL : 1;
#pragma unroll kUnroll
  for (int c = kFold ? ka : ka + 1; c <= kb + 1; ++c) {
    const Cons uC = src.load(c + 1);  // (a tight source hands over a preloaded cell)
    const bool upd = !kFold || c > ka;
    if (probe) {
      same = same_bits(uC, src.prev()) ? same + 1 : 0;
      saw |= same >= 5;
      // cells c-4..c+1 equal and the previous update the identity: cell c-1
      // keeps its input (see the comment above)
      if (__all_sync(0xffffffffu, (upd && same >= 5 && idprev) || !src.active)) {
        StepOut o;
        o.un = uC;  // == cell c-1, bit for bit
        o.fU = -1;
        o.fD = -1;
        o.spd = 0.0;  // cell c-2's equal speed is already in the maximum
        sink(c - 1, o);
        if (src.active) src.count_skip();
        src.boundary(c);
        if constexpr (Src::kTight) {
          // steady uniform run: the next cell repeats this one in every lane
          // -> the same shortcut, without the window bookkeeping (the
          // fused step's column phase); the first cell that differs goes
          // back to the general iteration, preloaded
          src.enter_tight(uC);
          while (c <= kb) {
            // a whole output chunk at once where the cursors sit on a chunk
            // boundary: its four incoming cells compared with one vote
            if (c + 3 <= kb && src.chunk_aligned() &&
                __all_sync(0xffffffffu, src.chunk_equal(uC) || !src.active)) {
              o.un = uC;  // the same bits
              src.take_chunk(sink, c, o);
              c += 4;
              same += 4;
              continue;
            }
            const Cons un = src.peek(c + 2);
            if (!__all_sync(0xffffffffu, same_bits(un, uC) || !src.active)) {
              src.preload(un);
              break;
            }
            ++c;
            ++same;
            o.un = un;
            sink(c - 1, o);
            if (src.active) src.count_skip();
            src.boundary(c);
          }
        }
        continue;
      }
    }
    StepOut o;
    step_cell<2, WANT_DT, FLUX>(m, w, uC, half, dtdx, spacing, g,
                                [&] { return src.reload(c - 1); }, o, memo, upd);
    if (o.fC >= 0) keep_min(ekey, key_base | ((unsigned long long)(c + 1 + kg) << 2) | o.fC);
    if (o.fR >= 0)
      keep_min(ekey, key_base | (1ull << 20) | ((unsigned long long)(c - 1 + kg) << 2) | o.fR);
    if (upd) {
      if (o.fU >= 0)
        keep_min(ekey, key_base | (2ull << 20) | ((unsigned long long)(c - 1 + kg) << 2) | o.fU);
      if (probe) {
        // only worth knowing where the next window can be uniform
        idprev = false;
        if (__any_sync(0xffffffffu, same >= 4))
          idprev = same >= 4 && o.fU < 0 && (!WANT_DT || o.fD < 0) &&
                   same_bits(o.un, src.reload(c - 1));
      }
      sink(c - 1, o);
    }
    src.boundary(c);
    w.wA = w.wB;
    w.wB = o.wC;
    w.frPrev = o.fr;
    w.fluxPrev = o.F;
  }
  if (kSkip) {
    if (!probe) --src.skip_cool;
    // (a warp without an active lane -- the fused step's last band -- has seen
    // nothing either way and keeps probing)
    else if (__any_sync(0xffffffffu, src.active) && !__any_sync(0xffffffffu, saw && src.active))
      src.skip_cool = kSkipCool;
  }
  // the memo carries over to this thread's next work item only if its
  // entries are exact: written by an exact pass, or by a fast pass that kept
  // every range (this lane's own flag -- masked lanes included)
  src.memo_valid = memo.valid && (!M::kFast || m.ok);
  return m.ok;
}

// The walker a work item runs.  HLLC: the fast pass of a warp that is probing
// for uniform windows runs the instantiation with the identity, every other
// pass (a cooling-down warp on dense flow, the redo pass) one without it --
// the compares and the shortcut's registers cost dense flow 5-8% otherwise.
// Exact-10: one instantiation with a run-time probe (its solver is ~5k
// instructions per copy; a second copy would not fit the instruction cache),
// and its uniform cells are memo hits anyway.
template <class M, bool WANT_DT, int FLUX, class Src, class Sink>
__device__ __forceinline__ bool walk_strip(int ka, int kb, Src& src, Sink& sink, const Gas& g,
                                           double dtdx, double spacing,
                                           unsigned long long key_base, int kg,
                                           unsigned long long& ekey) {
  if constexpr (FLUX == 1) {
    return walk_strip_impl<M, WANT_DT, FLUX, true>(ka, kb, src, sink, g, dtdx, spacing, key_base,
                                                   kg, ekey);
  } else if constexpr (!HB_SKIP || !M::kFast) {
    return walk_strip_impl<M, WANT_DT, FLUX, false>(ka, kb, src, sink, g, dtdx, spacing, key_base,
                                                    kg, ekey);
  } else {
    if (src.skip_cool == 0)
      return walk_strip_impl<M, WANT_DT, FLUX, true>(ka, kb, src, sink, g, dtdx, spacing, key_base,
                                                     kg, ekey);
    --src.skip_cool;
    return walk_strip_impl<M, WANT_DT, FLUX, false>(ka, kb, src, sink, g, dtdx, spacing, key_base,
                                                    kg, ekey);
  }
}

// Programmatic dependent launch (the sweeps are launched with
// cudaLaunchAttributeProgrammaticStreamSerialization): a sweep lets the next
// one be scheduled at once -- its CTAs occupy SM slots as this grid's retire
// and do their local setup -- and each sweep waits for its predecessor's
// completion before touching any global state.
__device__ __forceinline__ void pdl_wait() {
#if HB_PDL
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}
__device__ __forceinline__ void pdl_launch_dependents() {
#if HB_PDL
  asm volatile("griddepcontrol.launch_dependents;" :::);
#endif
}

// The warp's count of uniform-window cell updates -> the sweep's counter.
__device__ __forceinline__ void add_skipped(const SweepArgs& a, unsigned n) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
  if ((threadIdx.x & 31) == 0 && n && a.skipped) atomicAdd(a.skipped, (unsigned long long)n);
}

__device__ __forceinline__ bool latched(const SweepArgs& a) {
  return *(volatile unsigned long long*)a.err != kNoError;
}

__device__ __forceinline__ double step_dt(const SweepArgs& a) {
  return a.explicit_dt ? a.dt_value : a.cfl * __longlong_as_double((long long)*a.limit_in);
}

// Work distribution: a sweep is split into items of 32 strips x one segment
// of a.seg cells; the persistent warps of the launch claim items from an
// atomic counter (item = segment * groups + group, so neighbouring warps
// work on neighbouring strips).  Cells whose faces differ cost several times
// cells in uniform flow (HLLC vs the equal-state shortcut, :70-73), so
// dynamic claiming keeps all SMs busy when the active region is localised
// (shock tubes, blasts).  Each sweep resets the other sweep's counter for
// the next launch on the stream.
// Claim order: items run band by band, a band being `band` consecutive strip
// groups x all segments, segment-major inside the band (so neighbouring warps
// work on neighbouring strips).  The resident warps therefore stream through a
// compact part of the grid: on large grids a segment-major order over all
// strips (band >= groups) spreads the concurrent accesses of the row sweep
// over every grid row -- the whole state -- at once.
__device__ __forceinline__ void item_coords(int item, int groups, int nseg, int band, int& grp,
                                            int& sg) {
  const int per = band * nseg;
  const int b = item / per;
  const int r = item - b * per;
  const int rem = groups - b * band;
  const int gb = rem < band ? rem : band;  // the last band may be partial
  sg = r / gb;
  grp = b * band + (r - sg * gb);
}

__device__ __forceinline__ int claim(unsigned* counter) {
  int item = 0;
  if ((threadIdx.x & 31) == 0) item = (int)atomicAdd(counter, 1u);
  return __shfl_sync(0xffffffffu, item, 0);
}

#ifndef HB_PDL
#define HB_PDL 1
#endif
#ifndef HB_X_MINB
#define HB_X_MINB 4
#endif
#ifndef HB_Y_MINB
#ifdef HB_TOLERANCE
#define HB_Y_MINB 4  // 4-cell ring, 48 KB per CTA
#else
#define HB_Y_MINB 3  // the 8-cell ring (64 KB per CTA) allows 3 CTAs per SM anyway
#endif
#endif
#ifndef HB_EX_MINB  // exact-10 sweeps (long log/exp chains, ~200 registers)
#define HB_EX_MINB 3
#endif



// ---------------------------------------------------------------------------
// Row sweep with TMA-staged tiles, one independent pipeline per warp.

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  unsigned done = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!done);
}

__device__ __forceinline__ void tma_load5(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                          int c1, int c2, int c3, int c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
      : "memory");
}

__device__ __forceinline__ void tma_store5(const CUtensorMap* map, const void* src, int c0, int c1,
                                           int c2, int c3, int c4) {
  asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5, %6}], [%1];" ::
                   "l"(map),
               "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
               : "memory");
}

__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read1() {
  asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// TMA staging (both sweeps): a warp (one strip per lane) walks a segment in
// chunks of C = Staging<AXIS, FLUX>::C cells.  Chunk Q holds strip cells
// [ka-C+CQ, ka-1+CQ] of all four variables:
//   AXIS 1 (row sweep):    one box {C cols, 1 var, 32 rows} per variable,
//                          smem [var][row][col] (C = 8: 64-byte box rows,
//                          SWIZZLE_64B)
//   AXIS 0 (column sweep): one box {32 cols, 4 vars, C rows},
//                          smem [row][var][col]
// so a lane's cell is 8 bytes at stride 8C bytes (row sweep) or consecutive
// lanes read consecutive 8-byte words (column sweep).  Box rows are 64 or
// 256 bytes at 64-byte aligned addresses (kColOff): whole TMA fetch units,
// so no fetched byte is wasted.  A ring of NBUF buffers is used in place:
// once a cell has been read into registers its slot receives the updated
// cell (2 iterations later), and a completed chunk leaves with TMA
// bulk-tensor stores before its buffer is refilled.  With three buffers the
// refill goes to the buffer stored one chunk earlier (its store has long
// left shared memory); with two, the buffer just stored is refilled with the
// chunk after next once that store has read it out.  Chunk numbering runs on
// across the warp's items so buffer/phase bookkeeping never resets.

// The staged sweeps' dynamic shared memory (hb_smem, declared above):
// addressing it as hb_smem + offset (rather than through generic pointers)
// lets the compiler emit LDS/STS with 32-bit addresses.

template <int AXIS, int FLUX>
struct Tiles {
  static constexpr bool kTight = false;  // no tight uniform-run loop (walk_strip_impl)
  static constexpr int C = Staging<AXIS, FLUX>::C;
  static constexpr int NBUF = Staging<AXIS, FLUX>::NBUF;
  static constexpr int kChunkBytes = Staging<AXIS, FLUX>::kChunkBytes;
  static constexpr int kVarBytes = 32 * C * 8;  // row sweep: one variable of a chunk
  static_assert(NBUF >= 2 && NBUF <= 4, "ring of 2-4 buffers");
  // smem bytes between consecutive cells of a strip / adjacent strips
  // AXIS 0: one box {32 cols, C rows, 4 vars} per chunk, slot
  //   [var][pos][lane]; AXIS 1: one tiled block {C cols, 32 rows, 4 vars},
  //   slot [var][lane][pos].
  static constexpr uint32_t kPosBytes = 8 * (AXIS == 0 ? 32 : 1);
  static constexpr uint32_t kLaneBytes = AXIS == 0 ? 8 : C * 8;
  static constexpr uint32_t kVarStride = AXIS == 0 ? C * 32 * 8 : kVarBytes;

  const CUtensorMap* load_map;
  const CUtensorMap* store_map;
  uint32_t base;        // offset of this warp's NBUF consecutive kChunkBytes buffers
  uint32_t full;        // offset of this warp's NBUF mbarriers
  uint32_t memo_at;     // this thread's exact-10 interface memo (Memo)
  bool memo_valid;      // the memo holds an exact entry (kept across work items)
  int lane;
  int s0;               // first strip of the item: column j0 (AXIS 0) or row i0 (AXIS 1)
  int ka, kb;           // output strip cells
  int nq;               // chunks of this item (cells ka-C .. kb+2)
  unsigned q0;          // running chunk number of this item's chunk 0
  int T;                // next chunk to complete (flush)
  bool active;
  // Per-cell cursors (hb_smem offsets of this lane's variable-0 slot): the
  // next cell to load, and the cell being updated (reload + put).  The
  // walker visits cells in order, so they advance by one slot per cell
  // instead of recomputing chunk/buffer indices.
  uint32_t lo_addr, wr_addr;
  uint32_t last_addr, prev_addr;  // slots of the last two loaded cells (uniform-window test)
  unsigned nskip;       // cell updates taken by the uniform-window identity (this warp)
  int skip_cool;        // items left before this warp probes for uniform windows again
  uint32_t sw;          // this lane's TMA swizzle term (row sweep)
  int lo_pos, lo_buf, wr_pos, wr_buf;
  unsigned lo_par;      // mbarrier phase parity of the load cursor's buffer

  __device__ __forceinline__ static int chunks(int ka_, int kb_) {
    return (kb_ + 2 - (ka_ - C) + C) / C;
  }
  __device__ __forceinline__ uint8_t* buf(int q) {
    return hb_smem + base + ((q0 + q) % NBUF) * kChunkBytes;
  }
  __device__ __forceinline__ uint64_t* bar(int q) {
    return (uint64_t*)(hb_smem + full) + (q0 + q) % NBUF;
  }
  // Tensor coordinates {column offset, variable, plane row} of the chunk
  // whose first strip cell is k (cell k is grid index k-1 along the strip).
  __device__ __forceinline__ int c0(int k) const { return AXIS == 0 ? s0 + kColOff : k - 1 + kColOff; }
  __device__ __forceinline__ int c2(int k) const { return AXIS == 0 ? k : s0 + 1; }

  __device__ __forceinline__ void issue(int q) {  // lane 0 only
    if (q >= nq) return;
    mbar_expect_tx(bar(q), kChunkBytes);
    const int k = ka - C + q * C;
    if constexpr (AXIS == 0) {
      // U_a: 4 column blocks x grid rows k-1 .. k+2 (one block row; r + 1 =
      // grid row - 1 of the first row, >= -4) -> smem [var][row][col]
      const int r = k - 2;
      tma_load5(buf(q), load_map, bar(q), 0, c0(k) >> 3, r & 31, 0, (r >> 5) + 1);
    } else {
      // tiled U_b: the item's block row (s0 - 1) / 32, the chunk's column block
      const int col = c0(k);
      tma_load5(buf(q), load_map, bar(q), col & 7, col >> 3, 0, 0, (s0 + 31) >> 5);
    }
  }

  __device__ __forceinline__ void store(int t) {  // lane 0 only
    const int k = ka - C + t * C;
    if constexpr (AXIS == 0) {
      // tiled U_b: 4 column blocks x grid rows k-1 .. k+2 (one block row)
      const int r = k - 2;  // grid row - 1 of the chunk's first row (>= 0 for stored chunks)
      tma_store5(store_map, buf(t), 0, c0(k) >> 3, r & 31, 0, (r >> 5) + 1);
    } else {
      // U_a: one block (the item's block row, the chunk's column block)
      const int col = c0(k);
      tma_store5(store_map, buf(t), col & 7, col >> 3, 0, 0, (s0 + 31) >> 5);
    }
    bulk_commit();
  }

  // sweep orientation: mom_a is the momentum along the strip
  __device__ __forceinline__ Cons get(uint32_t at) const {
    constexpr int va = AXIS == 0 ? 1 : 2, vb = AXIS == 0 ? 2 : 1;
    const uint8_t* b = hb_smem + (at ^ sw);
    return {*(const double*)(b), *(const double*)(b + va * kVarStride),
            *(const double*)(b + vb * kVarStride), *(const double*)(b + 3 * kVarStride)};
  }

  // Cell k (= the load cursor's cell: ka-2, ka-1, ... in order).  Strips
  // past the grid compute on whatever the box holds (zero fill, ghost or
  // padding cells); their results, flags and errors are masked.
  __device__ __forceinline__ Cons load(int) {
    if (lo_pos == 0) mbar_wait((uint64_t*)(hb_smem + full) + lo_buf, lo_par);
    const Cons u = get(lo_addr);
    prev_addr = last_addr;
    last_addr = lo_addr;
    lo_addr += kPosBytes;
    if (++lo_pos == C) {
      lo_pos = 0;
      lo_addr += kChunkBytes - C * kPosBytes;
      if (++lo_buf == NBUF) {
        lo_buf = 0;
        lo_addr -= NBUF * kChunkBytes;
        lo_par ^= 1u;
      }
    }
    return u;
  }

  // The cell being updated, again (staged; its slot is overwritten only by put).
  __device__ __forceinline__ Cons reload(int) { return get(wr_addr); }

  // The cell loaded before the last one (its slot is rewritten only by the
  // update two iterations after its load, and its chunk is not flushed
  // before that).
  __device__ __forceinline__ Cons prev() const { return get(prev_addr); }
  __device__ __forceinline__ void count_skip() { ++nskip; }

  // The TMA swizzle term of strip (lane) l's slots: row sweep SWIZZLE_32B
  // (C = 4) flips the 16-byte half of a 32-byte row with address bit 7 (bit
  // 2 of the row); SWIZZLE_64B (C = 8) XORs the 16-byte unit index (bits 4-5)
  // with bits 7-8 (row bits 1-2); the column sweep is not swizzled.
  __device__ __forceinline__ static uint32_t swz(int l) {
    if constexpr (AXIS == 0) return 0u;
    return C == 4 ? (uint32_t)((l >> 2) & 1) << 4 : (uint32_t)((l >> 1) & 3) << 4;
  }

  // The cell being updated, of strip `ln` (default: this lane's), receives u.
  __device__ __forceinline__ void put(int, const Cons& u, int ln = -1) {
    constexpr int va = AXIS == 0 ? 1 : 2, vb = AXIS == 0 ? 2 : 1;
    uint8_t* b = hb_smem + (ln < 0 ? (wr_addr ^ sw)
                                   : ((wr_addr + (ln - lane) * (int)kLaneBytes) ^ swz(ln)));
    *(double*)(b) = u.r;
    *(double*)(b + va * kVarStride) = u.ma;
    *(double*)(b + vb * kVarStride) = u.mb;
    *(double*)(b + 3 * kVarStride) = u.e;
  }

  // After iteration c (cell c-1 updated for c > ka): advance the update
  // cursor; chunk boundaries fall on c - ka = C*T.
  __device__ __forceinline__ void boundary(int c) {
    if (c > ka) {
      wr_addr += kPosBytes;
      if (++wr_pos == C) {
        wr_pos = 0;
        wr_addr += kChunkBytes - C * kPosBytes;
        if (++wr_buf == NBUF) {
          wr_buf = 0;
          wr_addr -= NBUF * kChunkBytes;
        }
      }
    }
    if (c >= ka && wr_pos == 0) flush(T++);
  }

  // Chunk t's outputs are complete (the load cursor is 2 cells into chunk
  // t+1): store it and refill a free buffer.
  __device__ __forceinline__ void flush(int t) {
    if constexpr (NBUF == 2) {
      fence_async_smem();  // this lane's slot writes -> async proxy
      __syncwarp();
      if (lane == 0) {
        if (t >= 1) {
          store(t);
          bulk_wait_read0();  // chunk t's store has read its buffer
        }
        issue(t + 2);         // ... which now receives chunk t+2
      }
    } else {
      if (lane == 0) bulk_wait_read0();  // chunk t-1's stores have left smem
      fence_async_smem();
      __syncwarp();
      if (lane == 0) {
        if (t >= 1) store(t);
        issue(t + NBUF - 1);  // into the buffer of chunk t-1
      }
    }
  }

  // Stage the first chunks of an item (the first load is cell ka-2, slot C-2
  // of chunk 0; the first update is cell ka, slot 0 of chunk 1) / drain it.
  __device__ __forceinline__ void begin() {
    T = 0;
    const int b0 = (int)(q0 % NBUF), b1 = (b0 + 1) % NBUF;
    lo_buf = b0;
    lo_pos = C - 2;
    lo_par = (q0 / NBUF) & 1u;
    lo_addr = base + b0 * kChunkBytes + (C - 2) * kPosBytes + lane * kLaneBytes;
    last_addr = prev_addr = lo_addr;
    wr_buf = b1;
    wr_pos = 0;
    wr_addr = base + b1 * kChunkBytes + lane * kLaneBytes;
    if (lane == 0)
      for (int q = 0; q < (NBUF == 2 ? 2 : NBUF - 1); ++q) issue(q);
    mbar_wait((uint64_t*)(hb_smem + full) + lo_buf, lo_par);
  }
  __device__ __forceinline__ void end() {
    if (wr_pos != 0) flush(T);          // a short final chunk
    if (lane == 0) bulk_wait_read0();   // the ring is free again
    __syncwarp();
    q0 += nq;
  }
};

// Shared-memory carve-up of the staged sweeps: 4 warps x NBUF chunk
// buffers, then 4 x NBUF mbarriers (then the exact-10 memos).
template <int AXIS, int FLUX>
__device__ __forceinline__ Tiles<AXIS, FLUX> make_tiles(const CUtensorMap* load_map,
                                                        const CUtensorMap* store_map) {
  using Tl = Tiles<AXIS, FLUX>;
  // swizzle atoms repeat every 256 (32B) / 512 (64B) bytes
  const uint32_t pad = (1024u - (smem_u32(hb_smem) & 1023u)) & 1023u;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  Tl t;
  t.load_map = load_map;
  t.store_map = store_map;
  t.base = pad + warp * (Tl::NBUF * Tl::kChunkBytes);
  t.full = pad + 4 * Tl::NBUF * Tl::kChunkBytes + warp * Tl::NBUF * 8;
  t.memo_at = pad + 4 * Tl::NBUF * Tl::kChunkBytes + 4 * Tl::NBUF * 8 + threadIdx.x * 8;
  t.memo_valid = false;
  t.lane = lane;
  t.q0 = 0;
  t.nskip = 0;
  t.skip_cool = 0;
  t.sw = Tl::swz(lane);
  if (lane == 0) {
    for (int q = 0; q < Tl::NBUF; ++q) mbar_init((uint64_t*)(hb_smem + t.full) + q, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  return t;
}

// Column sweep with TMA-staged tiles (same pipeline as the row sweep).
template <int FLUX>
__global__ void __launch_bounds__(128, FLUX == 0 ? HB_X_MINB : HB_EX_MINB)
    sweep_x_tma_kernel(SweepArgs a, const __grid_constant__ CUtensorMap load_map,
                       const __grid_constant__ CUtensorMap store_map) {
  pdl_launch_dependents();
  auto t = make_tiles<0, FLUX>(&load_map, &store_map);
  const int lane = t.lane;
  const Gas g = make_gas(a.gamma);
  pdl_wait();
  if (latched(a)) return;
  if (*(volatile unsigned long long*)a.dt_err != kNoError) {
    // compute_dt of this step failed (detected by the previous row sweep).
    if (blockIdx.x == 0 && threadIdx.x == 0) record(a.err, *(volatile unsigned long long*)a.dt_err);
    return;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (a.limit_out) *a.limit_out = kEmptyLimit;
    *a.counter_next = 0u;
  }
  const double dtdx = step_dt(a) / a.dx;
  const size_t pitch = a.pitch;
  const int ny = a.ny;
  const bool refl = a.bc == 0;
  const int groups = (ny + 31) >> 5;
  const int items = groups * a.nseg;
  double* __restrict__ dst = a.dst;
  for (int item = claim(a.counter); item < items; item = claim(a.counter)) {
    int grp, sg;
    item_coords(item, groups, a.nseg, a.band, grp, sg);
    const int j0 = (grp << 5) + 1;
    const int j = j0 + lane;
    const bool active = j <= ny;
    const int i_lo = 1 + sg * a.seg;
    const int i_hi = min(a.nx, i_lo + a.seg - 1);
    t.s0 = j0;
    t.ka = i_lo + 1;
    t.kb = i_hi + 1;
    t.nq = t.chunks(t.ka, t.kb);
    t.active = active;
    // warps holding a y-wall column (1, 2, ny-1 or ny) write the ghost columns
    const bool edge = grp == 0 || (grp << 5) + 32 >= ny - 1;
    const unsigned long long base = error_key(a.step, 1, j, 0, 0, 0);
    auto pass = [&](auto math) {
      using M = decltype(math);
      t.begin();
      // ghost columns of U_b (tiled): inside this warp's store box (its 32
      // columns) a ghost goes into the slot of the lane that holds that
      // column -- an inactive lane, whose slot the TMA store writes -- else
      // straight to memory (a block no store box covers)
      auto put = [&](int k, int i, int jt, const Cons& u, bool neg) {
        Cons gh = u;
        if (neg) gh.mb = -gh.mb;
        const int d = jt - j0;
        if (d >= 0 && d < 32) {
          t.put(k, gh, d);
          return;
        }
        // a column inside another warp's store box (reflecting walls with
        // ny % 32 == 1: ghost ny+2 mirrors column ny-1 of the previous group)
        // is written after the sweep by ghost_fix_kernel
        if (jt > ny && ((jt - 1) >> 5) < groups) return;
        double* q = dst + cell_index(pitch, 0, i, jt);
        q[0] = gh.r;
        q[kVarStep] = gh.ma;
        q[2 * kVarStep] = gh.mb;
        q[3 * kVarStep] = gh.e;
      };
      auto sink = [&](int k, const StepOut& o) {
        if (active) t.put(k, o.un);
        if (edge && active) {  // y-wall ghosts of the column-sweep output (grid.cpp:44-59)
          const int i = k - 1;
          if (refl) {
            if (j <= 2) put(k, i, 1 - j, o.un, true);
            if (j >= ny - 1) put(k, i, 2 * ny + 1 - j, o.un, true);
          } else {
            if (j == 1) { put(k, i, 0, o.un, false); put(k, i, -1, o.un, false); }
            if (j == ny) { put(k, i, ny + 1, o.un, false); put(k, i, ny + 2, o.un, false); }
          }
        }
      };
      unsigned long long ek = kNoError;
      const bool ok = walk_strip<M, false, FLUX>(t.ka, t.kb, t, sink, g, dtdx, 0.0, base, a.row0, ek);
      t.end();
      return make_pair_ok(ok, ek);
    };
    OkKey r = pass(FastMath{});
    if (!__all_sync(0xffffffffu, r.ok || !active)) {
      if (lane == 0) bulk_wait0();  // the fast pass's stores have landed
      __syncwarp();
      r = pass(ExactMath{});
    }
    if (active && r.key != kNoError) record(a.err, r.key);
  }
  if (lane == 0) bulk_wait0();
  add_skipped(a, t.nskip);
}

// PEER: also store the halo rows into the neighbours' inboxes (peer-memory
// halo; a separate instantiation keeps the single-GPU path unchanged).
template <int FLUX, bool PEER>
__global__ void __launch_bounds__(128, FLUX == 0 ? HB_Y_MINB : HB_EX_MINB) sweep_y_kernel(SweepArgs a,
                                                       const __grid_constant__ CUtensorMap load_map,
                                                       const __grid_constant__ CUtensorMap store_map) {
  pdl_launch_dependents();
  auto t = make_tiles<1, FLUX>(&load_map, &store_map);
  const int lane = t.lane;
  const Gas g = make_gas(a.gamma);
  pdl_wait();
  if (latched(a)) return;
  if (blockIdx.x == 0 && threadIdx.x == 0) *a.counter_next = 0u;
  const double dtdx = step_dt(a) / a.dx;
  const size_t pitch = a.pitch;
  const int nx = a.nx;
  const bool refl = a.bc == 0;
  const int groups = (nx + 31) >> 5;
  const int items = groups * a.nseg;
  double* __restrict__ dst = a.dst;
  double spd_max = 0.0;  // speeds are >= +0
  unsigned long long dt_key = kNoError;
  bool wrote_peer = false;

  for (int item = claim(a.counter); item < items; item = claim(a.counter)) {
    int grp, sg;
    item_coords(item, groups, a.nseg, a.band, grp, sg);
    const int i0 = (grp << 5) + 1;
    const int i = i0 + lane;
    const bool active = i <= nx;
    const int j_lo = 1 + sg * a.seg;
    const int j_hi = min(a.ny, j_lo + a.seg - 1);
    t.s0 = i0;
    t.ka = j_lo + 1;
    t.kb = j_hi + 1;
    t.nq = t.chunks(t.ka, t.kb);
    t.active = active;
    // warps holding x-wall rows write the ghost rows of the next step
    const bool mirror_lo = a.wall_lo && grp == 0;
    const bool mirror_hi = a.wall_hi && (grp << 5) + 32 >= nx - 1;  // rows nx-1, nx
    // peer-memory halo: rows 1..2 / nx-1..nx also go to the neighbours' inboxes
    const bool send_up = PEER && a.halo_up && grp == 0;
    const bool send_dn = PEER && a.halo_dn && (grp << 5) + 32 >= nx - 1;
    wrote_peer |= send_up | send_dn;
    // this lane's row has ghost-row or halo copies to write (rare lanes only:
    // the per-cell test is one predicate)
    const bool extra = active && (((mirror_lo || send_up) && i <= 2) ||
                                  ((mirror_hi || send_dn) && i >= nx - 1));
    const int gi = a.row0 + i;
    const unsigned long long base = error_key(a.step, 2, gi, 0, 0, 0);
    // x-wall ghost rows of U_a: inside this warp's store blocks (its 32 rows)
    // a ghost row goes into the slot of the lane that holds that row -- an
    // inactive lane, whose slot the TMA store writes -- else straight to
    // memory (block row -1 and rows no store block covers); a row inside
    // another warp's blocks (reflecting walls with nx % 32 == 1: ghost nx+2
    // mirrors row nx-1 of the previous group) is written after the sweep by
    // ghost_fix_kernel
    auto put_row = [&](int k, int ii, int j, const Cons& u, bool neg) {
      Cons gh = u;
      if (neg) gh.mb = -gh.mb;  // sweep orientation: mom_b is mom_x
      const int d = ii - i0;
      if (d >= 0 && d < 32) {
        t.put(k, gh, d);
        return;
      }
      if (ii > nx && ((ii - 1) >> 5) < groups) return;
      double* q = dst + cell_index(pitch, 0, ii, j);
      q[0] = gh.r;
      q[kVarStep] = gh.mb;
      q[2 * kVarStep] = gh.ma;
      q[3 * kVarStep] = gh.e;
    };
    auto put_peer = [&](double* q, const Cons& u) {  // NVLink store into a peer's inbox
      q[0] = u.r;
      q[2 * pitch] = u.ma;
      q[pitch] = u.mb;
      q[3 * pitch] = u.e;
    };
    double spd_item;
    unsigned long long dt_item;
    // One pass over the item with math policy M (tiles restaged from U_b).
    auto pass = [&](auto math) {
      using M = decltype(math);
      spd_item = 0.0;
      dt_item = kNoError;
      t.begin();
      auto sink = [&](int k, const StepOut& o) {
        t.put(k, o.un);
        const int j = k - 1;
        if (extra) {
        if (mirror_lo && active && i <= 2) {  // x-wall ghosts for the next column sweep (grid.cpp:26-42)
          if (refl) put_row(k, 1 - i, j, o.un, true);
          else if (i == 1) { put_row(k, 0, j, o.un, false); put_row(k, -1, j, o.un, false); }
        }
        if (mirror_hi && active && i >= nx - 1) {
          if (refl) put_row(k, 2 * nx + 1 - i, j, o.un, true);
          else if (i == nx) { put_row(k, nx + 1, j, o.un, false); put_row(k, nx + 2, j, o.un, false); }
        }
        if constexpr (PEER) {
          if (send_up && active && i <= 2)  // -> upper neighbour's ghost rows nx'+1..nx'+2
            put_peer(a.halo_up + (size_t)(i - 1) * 4 * pitch + (j + kColOff), o.un);
          if (send_dn && active && i >= nx - 1)  // -> lower neighbour's ghost rows -1..0
            put_peer(a.halo_dn + (size_t)(i - (nx - 1)) * 4 * pitch + (j + kColOff), o.un);
        }
        }
        if (a.want_limit) {
          if (o.fD >= 0) keep_min(dt_item, error_key(a.step + 1, 0, gi, 0, j, o.fD));
          else spd_item = smax(spd_item, o.spd);
        }
      };
      unsigned long long ek = kNoError;
      // the signal speeds are evaluated even when no limit is wanted (the last
      // step of a run, advance): one walker instantiation per math policy
      // keeps the kernel's code within the instruction cache
      const bool ok = walk_strip<M, true, FLUX>(t.ka, t.kb, t, sink, g, dtdx, a.spacing, base, 0, ek);
      t.end();
      return make_pair_ok(ok, ek);
    };
    OkKey r = pass(FastMath{});
    // a fast path left its proven range somewhere: the warp redoes the item
    // with the exact policy (restaging and overwriting all): the compiler's
    // IEEE division/sqrt in the bitwise TU; in the tolerance TU the same
    // formulas as the fast pass wherever their operands are in range and IEEE
    // outside it, with the reference's branches and error reports
    if (!__all_sync(0xffffffffu, r.ok || !active)) {
      if (lane == 0) bulk_wait0();  // the fast pass's stores have landed
      __syncwarp();
      r = pass(ExactMath{});
    }
    if (active) {
      if (r.key != kNoError) record(a.err, r.key);
      keep_min(dt_key, dt_item);
      spd_max = smax(spd_max, spd_item);
    }
  }
  if (lane == 0) bulk_wait0();
  add_skipped(a, t.nskip);
  // peer stores performed system-wide before this kernel completes (the
  // neighbour reads them after the dt allreduce that follows on the stream)
  if (PEER && wrote_peer) __threadfence_system();
  if (a.want_limit) {
    // largest speed of the warp (non-negative doubles order like their bits)
    // -> its cell_dt_limit, the warp's minimum limit
    const double smx = __longlong_as_double(
        (long long)~warp_min_u64(~(unsigned long long)__double_as_longlong(spd_max)));
    const unsigned long long e = warp_min_u64(dt_key);
    if (lane == 0) {
      atomicMin(a.limit_out, (unsigned long long)__double_as_longlong(a.spacing / smx));
      if (e != kNoError) atomicMin(a.dt_err, e);
    }
  }
}

// The fused step (FUSED schedule): column and row sweep in one launch.
#include "hydro_fused.cuh"

// ---------------------------------------------------------------------------
// Start-of-run pass: apply_boundary on the physical walls of the current
// state and compute_dt's min-reduction for the first step.
__global__ void __launch_bounds__(256) HB_SWEEP(prologue_kernel)(PrologueArgs a) {
  const int j = 1 + blockIdx.x * blockDim.x + threadIdx.x;
  const bool active = j <= a.ny;
  const size_t pitch = a.pitch;
  double* u = a.u;
  const bool refl = a.bc == 0;
  const Gas g = make_gas(a.gamma);
  double lim = __longlong_as_double(0x7ff0000000000000ll);
#ifdef HB_TOLERANCE
  double spd = 0.0;  // the largest signal speed (speeds are >= +0)
#endif
  unsigned long long key = kNoError;
  const int nx = a.nx, ny = a.ny;
  for (int i = 1 + blockIdx.y; active && i <= nx; i += gridDim.y) {
    Cons c = {u[cell_index(pitch, 0, i, j)], u[cell_index(pitch, 1, i, j)],
              u[cell_index(pitch, 2, i, j)], u[cell_index(pitch, 3, i, j)]};
    auto put = [&](int ii, int jj, int negv) {
      u[cell_index(pitch, 0, ii, jj)] = c.r;
      u[cell_index(pitch, 1, ii, jj)] = negv == 1 ? -c.ma : c.ma;
      u[cell_index(pitch, 2, ii, jj)] = negv == 2 ? -c.mb : c.mb;
      u[cell_index(pitch, 3, ii, jj)] = c.e;
    };
    if (a.wall_lo && i <= 2) {
      if (refl) put(1 - i, j, 1);
      else if (i == 1) { put(0, j, 0); put(-1, j, 0); }
    }
    if (a.wall_hi && i >= nx - 1) {
      if (refl) put(2 * nx + 1 - i, j, 1);
      else if (i == nx) { put(nx + 1, j, 0); put(nx + 2, j, 0); }
    }
    if (a.full_bc) {
      if (refl) {
        if (j <= 2) put(i, 1 - j, 2);
        if (j >= ny - 1) put(i, 2 * ny + 1 - j, 2);
      } else {
        if (j == 1) { put(i, 0, 0); put(i, -1, 0); }
        if (j == ny) { put(i, ny + 1, 0); put(i, ny + 2, 0); }
      }
    }
    if (a.want_limit) {
#ifdef HB_TOLERANCE
      // the row sweep's dt speed (cell_speed == its epilogue's dt_speed)
      double sp;
      FastMath fm;
      int f = cell_speed(fm, c, g, sp);
      if (!fm.ok) {
        ExactMath em;
        f = cell_speed(em, c, g, sp);
      }
      if (f >= 0) {
        const unsigned long long k = error_key(a.step, 0, a.row0 + i, 0, j, f);
        key = k < key ? k : key;
      } else {
        spd = smax(spd, sp);
      }
#else
      double l;
      FastMath fm;
      int f = dt_limit(fm, c, fm.recip(c.r), a.spacing, g, l);
      if (!fm.ok) {
        ExactMath em;
        f = dt_limit(em, c, em.recip(c.r), a.spacing, g, l);
      }
      if (f >= 0) {
        const unsigned long long k = error_key(a.step, 0, a.row0 + i, 0, j, f);
        key = k < key ? k : key;
      } else {
        lim = smin(lim, l);
      }
#endif
    }
  }
  if (a.want_limit) {
#ifdef HB_TOLERANCE
    // largest speed of the warp -> spacing / speed, as the row sweep does
    const double smx = __longlong_as_double(
        (long long)~warp_min_u64(~(unsigned long long)__double_as_longlong(spd)));
    if (smx > 0.0) lim = a.spacing / smx;
#endif
    const unsigned long long m = warp_min_u64((unsigned long long)__double_as_longlong(lim));
    const unsigned long long e = warp_min_u64(key);
    if ((threadIdx.x & 31) == 0) {
      atomicMin(a.limit_out, m);
      if (e != kNoError) atomicMin(a.err, e);
    }
  }
}

#ifndef HB_TOLERANCE
// The one ghost column of the tiled U_b the column sweep cannot store: with
// reflecting walls and ny % 32 == 1, ghost column ny+2 (the mirror of column
// ny-1, grid.cpp:44-59) lies in the last column group's store box while its
// source column belongs to the previous group.
__global__ void ghost_fix_kernel(double* __restrict__ b, size_t pitch, int nx, int ny) {
  const int i = 1 + blockIdx.x * blockDim.x + threadIdx.x;
  if (i > nx) return;
  for (int v = 0; v < 4; ++v) {
    const double x = b[cell_index(pitch, v, i, ny - 1)];
    b[cell_index(pitch, v, i, ny + 2)] = v == 2 ? -x : x;
  }
}

// The same for U_a after a row sweep: with a reflecting lower wall and
// nx % 32 == 1, ghost row nx+2 (the mirror of row nx-1, grid.cpp:26-42) lies
// in the last row group's store blocks.
__global__ void ghost_row_fix_kernel(double* __restrict__ a, size_t pitch, int nx, int ny) {
  const int j = 1 + blockIdx.x * blockDim.x + threadIdx.x;
  if (j > ny) return;
  for (int v = 0; v < 4; ++v) {
    const double x = a[cell_index(pitch, v, nx - 1, j)];
    a[cell_index(pitch, v, nx + 2, j)] = v == 1 ? -x : x;
  }
}

// Row-layout rows <-> the tiled state.  rows[r * row_stride + (j + 1)] is
// cell (i0 + r, j), j = -1 .. ny+2, of variable v (the host Grid2D plane
// format, through the transfers' device staging); v = -1: all four
// variables of 2 rows in the halo-block format (element (r, v, j) at
// (4 r + v) pitch + j + kColOff, the inbox layout the row sweep's peer stores
// use).
__global__ void rows_tiles_kernel(double* rows, size_t row_stride, double* u, size_t pitch, int v,
                                  int i0, int n, int ny, int to_tiles) {
  const int j = -1 + (int)(blockIdx.x * blockDim.x + threadIdx.x);
  if (j > ny + 2) return;
  for (int r = blockIdx.y; r < n; r += gridDim.y) {
    for (int w = (v < 0 ? 0 : v); w <= (v < 0 ? 3 : v); ++w) {
      double* h = v < 0 ? rows + ((size_t)4 * r + w) * pitch + (j + kColOff)
                        : rows + (size_t)r * row_stride + (j + 1);
      double* d = u + cell_index(pitch, w, i0 + r, j);
      if (to_tiles) *d = *h;
      else *h = *d;
    }
  }
}

// compare_tolerance's max |a - b| / max(|a|, |b|, 1) over the interior
// (proj/src/audit.cpp:137-154) of two states of one geometry, as the bits of
// a non-negative double (atomicMax).
__global__ void compare_kernel(const double* __restrict__ a, const double* __restrict__ b,
                               size_t pitch, int nx, int ny, unsigned long long* out) {
  double m = 0.0;
  const size_t cells = (size_t)nx * ny;
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < 4 * cells;
       t += (size_t)gridDim.x * blockDim.x) {
    const int v = (int)(t / cells);
    const size_t c = t % cells;
    const int i = 1 + (int)(c / ny), j = 1 + (int)(c % ny);
    const size_t k = cell_index(pitch, v, i, j);
    const double x = a[k], y = b[k];
    const double r = fabs(x - y) / fmax(fmax(fabs(x), fabs(y)), 1.0);
    m = (r > m || r != r) ? r : m;  // a NaN difference propagates
  }
  unsigned long long bits = (unsigned long long)__double_as_longlong(m);
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long w = __shfl_xor_sync(0xffffffffu, bits, o);
    bits = w > bits ? w : bits;
  }
  if ((threadIdx.x & 31) == 0) atomicMax(out, bits);
}

// End-of-run ghosts: the reference's last apply_boundary ran on the column
// sweep output, so every ghost band mirrors U_b (grid.cpp:23-60).
__global__ void finish_kernel(FinishArgs a) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const size_t pitch = a.pitch;
  const bool refl = a.bc == 0;
  if (t < a.ny) {  // i-wall ghost rows from U_b interior rows
    const int j = t + 1;
    for (int layer = 1; layer <= 2; ++layer) {
      const int srcs[2] = {refl ? layer : 1, refl ? a.nx + 1 - layer : a.nx};
      const int gh[2] = {1 - layer, a.nx + layer};
      const int on[2] = {a.wall_lo, a.wall_hi};
      for (int s = 0; s < 2; ++s) {
        if (!on[s]) continue;
        for (int v = 0; v < 4; ++v) {
          const double x = a.post_x[cell_index(pitch, v, srcs[s], j)];
          a.u[cell_index(pitch, v, gh[s], j)] = (refl && v == 1) ? -x : x;
        }
      }
    }
  } else if (t < a.ny + a.nx) {  // j-wall ghost columns, already mirrored in U_b
    const int i = t - a.ny + 1;
    const int cols[4] = {-1, 0, a.ny + 1, a.ny + 2};
    for (int c = 0; c < 4; ++c)
      for (int v = 0; v < 4; ++v)
        a.u[cell_index(pitch, v, i, cols[c])] = a.post_x[cell_index(pitch, v, i, cols[c])];
  }
}

// ---------------------------------------------------------------------------
// Case initialisers (cases.cpp:11-69 and the BASELINE configs), bitwise equal
// to the host versions in hydro_host.cpp.
__device__ __forceinline__ unsigned long long splitmix64(unsigned long long x) {
  unsigned long long z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ double rnd_sym(unsigned long long seed, unsigned long long cell,
                                          int var) {
  const unsigned long long h = splitmix64(seed ^ (4ull * cell + (unsigned long long)var));
  const double unit = (double)(h >> 11) * 0x1.0p-53;
  return 2.0 * unit - 1.0;
}

__global__ void init_kernel(InitArgs a) {
  const int j = 1 + blockIdx.x * blockDim.x + threadIdx.x;
  if (j > a.ny) return;
  for (int i = 1 + blockIdx.y; i <= a.nx; i += gridDim.y) {
    const int gi = a.row0 + i;
    Prim w = {1.0, 0.0, 0.0, 1.0};
    switch (a.case_id) {
      case 1: w.p = 1e-5 * (a.gamma - 1.0); break;
      case 3: w.p = 1e-5; break;
      case 2:
        if (!(j <= a.ny / 2)) w = {0.125, 0.0, 0.0, 0.1};
        break;
      case 4:
        if (!(gi <= a.global_nx / 2)) w = {0.125, 0.0, 0.0, 0.1};
        break;
      case 5: {
        const unsigned long long cell =
            (unsigned long long)(gi - 1) * (unsigned long long)a.ny + (unsigned long long)(j - 1);
        w.r = 1.0 + 0.1 * rnd_sym(a.seed, cell, 0);
        w.p = 1.0 + 0.1 * rnd_sym(a.seed, cell, 1);
        w.va = 0.1 * rnd_sym(a.seed, cell, 2);
        w.vb = 0.1 * rnd_sym(a.seed, cell, 3);
        break;
      }
      default: break;
    }
    // prim_to_cons (euler_kernel.cpp:22-28)
    double e = w.p / (a.gamma - 1.0) + 0.5 * w.r * (w.va * w.va + w.vb * w.vb);
    if (a.case_id == 3 && gi == 1 && j == 1) e = 1.0 / (a.dx * a.dy);
    if (a.case_id == 1) {
      const int gnx = a.global_nx, ny = a.ny;
      const bool ci = (gnx % 2) ? (gi == (gnx + 1) / 2) : (gi == gnx / 2 || gi == gnx / 2 + 1);
      const bool cj = (ny % 2) ? (j == (ny + 1) / 2) : (j == ny / 2 || j == ny / 2 + 1);
      if (ci && cj) {
        const double share = 1.0 / ((double)((gnx % 2) ? 1 : 2) * (double)((ny % 2) ? 1 : 2));
        e = share / (a.dx * a.dy);
      }
    }
    const size_t p = a.pitch;
    a.u[cell_index(p, 0, i, j)] = w.r;
    a.u[cell_index(p, 1, i, j)] = w.r * w.va;
    a.u[cell_index(p, 2, i, j)] = w.r * w.vb;
    a.u[cell_index(p, 3, i, j)] = e;
  }
}

// ---------------------------------------------------------------------------
// Device-side audit: per-row FNV-1a hashes (the building block of the
// composable state hash, see hydro_gpu_state_hash) and per-row sums of one
// variable (fixed serial order: deterministic), one thread per (variable,
// row).  The reference's digest (audit.cpp:53-76) is byte-serial over the
// whole grid and stays a host step.
__global__ void row_audit_kernel(const double* __restrict__ u, size_t pitch, int nx, int ny,
                                 unsigned long long* __restrict__ hashes,
                                 double* __restrict__ sums) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= 4 * nx) return;
  const int v = t / nx, i = t % nx + 1;
  unsigned long long h = 14695981039346656037ull;
  double sum = 0.0;
  for (int j = 0; j < ny; ++j) {
    const double x = __ldg(u + cell_index(pitch, v, i, j + 1));
    const unsigned long long bits = (unsigned long long)__double_as_longlong(x);
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      h ^= (bits >> (8 * b)) & 0xffull;
      h *= 1099511628211ull;
    }
    sum += x;
  }
  hashes[t] = h;
  sums[t] = sum;
}

// FastMath against the compiler's IEEE operations (tests/test_gpu_math.py).
__global__ void math_selftest_kernel(int op, const double* a, const double* b, double* fast,
                                     double* ref, int* okv, size_t n) {
  const size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (t >= n) return;
  FastMath fm;
  if (op == 0) {  // general quotient (any signs)
    fast[t] = fm.divnf(a[t], b[t]);
    ref[t] = a[t] / b[t];
  } else if (op == 4) {  // density quotient (zero numerators, positive denominators)
    fast[t] = fm.divf(a[t], b[t]);
    ref[t] = a[t] / b[t];
  } else if (op == 5) {  // envelope-bounded quotient (divb: no range test)
    fast[t] = fm.divb(a[t], fm.recip(b[t]));
    ref[t] = a[t] / b[t];
  } else if (op == 2) {
    fast[t] = fm.divz(a[t], b[t]);
    ref[t] = a[t] / b[t];
  } else if (op == 3) {  // minmod of the differences (a, b)
    fast[t] = minmod_d_fast(a[t], b[t]);
    ref[t] = minmod_d(a[t], b[t]);
  } else {
    fast[t] = fm.sqrt(a[t]);
    ref[t] = sqrt(a[t]);
  }
  okv[t] = fm.ok ? 1 : 0;
}

#endif  // !HB_TOLERANCE

// Segment length for the persistent sweeps: about kItemsPerWarp work items
// per resident warp (dynamic balance), 16..128 cells, whole row-sweep chunks.
constexpr int kItemsPerWarp = 8;
int pick_seg(int n, int strips, int warps, int chunk, int items_per_warp = kItemsPerWarp,
             int max_seg = 128) {
  const long long groups = (strips + 31) / 32;
  long long segs = (long long)warps * items_per_warp / (groups > 0 ? groups : 1);
  if (segs < 1) segs = 1;
  long long seg = (n + segs - 1) / segs;
  if (seg < 16) seg = 16;
  if (seg > max_seg) seg = max_seg;
  seg = (seg + chunk - 1) / chunk * chunk;
  // small grids: 16-cell segments leave warps without work, and a segment
  // is a sequential walk, so trade halo recomputation for parallelism --
  // segments down to one chunk, about one item per resident warp
  if (groups * ((n + seg - 1) / seg) < warps) {
    long long s2 = (long long)n * groups / (warps > 0 ? warps : 1) / chunk * chunk;
    seg = s2 < chunk ? chunk : s2;
  }
  return (int)seg;
}

// Band width of the claim order (item_coords): band <= 0 picks about two
// bands' worth of items per wave of resident warps (the resident warps then
// touch ~2 x warps/nseg strip groups at a time), band > 0 is an override
// (>= groups: segment-major over all strips).
int pick_band(int band, int strips, int nseg, int warps, int div = 2) {
  const int groups = (strips + 31) / 32;
  if (band > 0) return band < groups ? band : groups;
  long long b = ((long long)warps + nseg - 1) / nseg;
  b = (b + div - 1) / div;
  if (b < 1) b = 1;
  return (int)(b < groups ? b : groups);
}

}  // namespace

int HB_SWEEP(query_geometry)(Geometry* g) {
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&g->sms, cudaDevAttrMultiProcessorCount, dev);
  cudaFuncSetAttribute(sweep_y_kernel<0, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kYSmemBytes);
  cudaFuncSetAttribute(sweep_y_kernel<1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kExYSmemBytes);
  cudaFuncSetAttribute(sweep_y_kernel<0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kYSmemBytes);
  cudaFuncSetAttribute(sweep_y_kernel<1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kExYSmemBytes);
  int ox = 0, oy = 0, ox1 = 0, oy1 = 0;
  cudaFuncSetAttribute(sweep_x_tma_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, kXSmemBytes);
  cudaFuncSetAttribute(sweep_x_tma_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kExXSmemBytes);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ox, sweep_x_tma_kernel<0>, 128, kXSmemBytes);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ox1, sweep_x_tma_kernel<1>, 128, kExXSmemBytes);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&oy, sweep_y_kernel<0, false>, 128, kYSmemBytes);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&oy1, sweep_y_kernel<1, false>, 128, kExYSmemBytes);
  g->ctas_x_per_sm = ox > 0 ? ox : 1;
  g->ctas_y_per_sm = oy > 0 ? oy : 1;
  g->ctas_x_exact = ox1 > 0 ? ox1 : 1;
  g->ctas_y_exact = oy1 > 0 ? oy1 : 1;
  int oxy = 0;
  cudaFuncSetAttribute(sweep_xy_kernel<0, false, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, kFSmemBytes);
  cudaFuncSetAttribute(sweep_xy_kernel<1, false, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, kFSmemBytes);
  cudaFuncSetAttribute(sweep_xy_kernel<0, true, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, kFSmemBytes);
  cudaFuncSetAttribute(sweep_xy_kernel<1, true, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, kFSmemBytes);
  cudaFuncSetAttribute(sweep_xy_kernel<0, false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kFSmemBytesEx);
  cudaFuncSetAttribute(sweep_xy_kernel<1, false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kFSmemBytesEx);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&oxy, sweep_xy_kernel<0, false, 0>, 256, kFSmemBytes);
  g->ctas_xy_per_sm = oxy > 0 ? oxy : 1;
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

#ifndef HB_TOLERANCE
bool make_tma_maps(TmaMaps* maps, double* A, double* B, size_t pitch, int nx, int ny) {
  (void)ny;
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return false;
    encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  }
  // a tiled state buffer (cell_index) as dims {column in block, column
  // block, row in block, var, block row}: strides not increasing, so a box
  // lands in smem as [var][row][block][column]
  const cuuint64_t ntj = pitch / 8;
  const cuuint64_t dim[5] = {8, ntj, 32, 4, (cuuint64_t)tile_rows(nx)};
  const cuuint64_t str[4] = {8192, 64, 2048, 8192 * ntj};
  auto enc = [&](CUtensorMap* m, double* base, const cuuint32_t* box, CUtensorMapSwizzle swz) {
    const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    return encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, base, dim, str, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  };
  constexpr int CX = Staging<0>::C, CY = Staging<1>::C, CE = Staging<1, 1>::C;
  const cuuint32_t box_x[5] = {8, 4, (cuuint32_t)CX, 4, 1};  // 32 columns x CX rows x 4 vars
  const cuuint32_t box_y[5] = {(cuuint32_t)CY, 1, 32, 4, 1};  // C columns x 32 rows x 4 vars
  const cuuint32_t box_ey[5] = {(cuuint32_t)CE, 1, 32, 4, 1};
  // row sweep: 64-byte (32-byte) box rows swizzled against the smem bank
  // conflicts of lane-per-row accesses; column sweep: lanes read consecutive
  // words
  auto swz = [](int c) { return c == 4 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_64B; };
  const CUtensorMapSwizzle none = CU_TENSOR_MAP_SWIZZLE_NONE;
  maps->y_cols = CY;
  maps->ey_cols = CE;
  // fused step: the column phase's 4-row chunks of a band (+ one block either
  // side) -> smem [var][row][col]; the row phase stores one row of one
  // variable (the band's kFW columns, 960 contiguous bytes of smem) per box
  const cuuint32_t box_fl[5] = {8, (cuuint32_t)kFLoadBlocks, 4, 4, 1};
  const cuuint32_t box_fs[5] = {8, (cuuint32_t)(kFW / 8), 1, 1, 1};
  if (!(enc(&maps->fa_load, A, box_fl, none) && enc(&maps->fb_load, B, box_fl, none) &&
        enc(&maps->fa_store, A, box_fs, none) && enc(&maps->fb_store, B, box_fs, none)))
    return false;
  return enc(&maps->x_load, A, box_x, none) && enc(&maps->x_store, B, box_x, none) &&
         enc(&maps->y_load, B, box_y, swz(CY)) && enc(&maps->y_store, A, box_y, swz(CY)) &&
         enc(&maps->ey_load, B, box_ey, swz(CE)) && enc(&maps->ey_store, A, box_ey, swz(CE));
}

#endif  // !HB_TOLERANCE

namespace {
template <class... KArgs, class... Args>
void launch_sweep_block(void (*kernel)(KArgs...), int ctas, int block, int smem, cudaStream_t s,
                        Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(ctas);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = HB_PDL;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kernel, args...);
}
template <class... KArgs, class... Args>
void launch_sweep(void (*kernel)(KArgs...), int ctas, int smem, cudaStream_t s, Args... args) {
  launch_sweep_block(kernel, ctas, 128, smem, s, args...);
}
}  // namespace

void HB_SWEEP(launch_sweep_x)(const SweepArgs& a0, const TmaMaps& maps, const Geometry& geo,
                    cudaStream_t s) {
  SweepArgs a = a0;
  const int ctas = geo.sms * (a.flux == 1 ? geo.ctas_x_exact : geo.ctas_x_per_sm);
  const int C = Staging<0>::C;
  if (a.seg <= 0) a.seg = pick_seg(a.nx, a.ny, ctas * 4, C);
  a.seg = (a.seg + C - 1) / C * C;  // chunks never straddle segments
  a.nseg = (a.nx + a.seg - 1) / a.seg;
  a.band = pick_band(a.band, a.ny, a.nseg, ctas * 4);
  if (a.flux == 1)
    launch_sweep(sweep_x_tma_kernel<1>, ctas, kExXSmemBytes, s, a, maps.x_load, maps.x_store);
  else
    launch_sweep(sweep_x_tma_kernel<0>, ctas, kXSmemBytes, s, a, maps.x_load, maps.x_store);
}

void HB_SWEEP(launch_sweep_y)(const SweepArgs& a0, const TmaMaps& maps, const Geometry& geo,
                    cudaStream_t s) {
  SweepArgs a = a0;
  const int ctas = geo.sms * (a.flux == 1 ? geo.ctas_y_exact : geo.ctas_y_per_sm);
  const int C = a.flux == 1 ? Staging<1, 1>::C : Staging<1>::C;
  // row sweep (HLLC): segments of at most 64 cells in narrow bands of row
  // groups -- the resident warps then read neighbouring 64-byte pieces of the
  // same grid rows (config 3 -4%, config 2 -4%, config 4 +1..3%)
  if (a.seg <= 0)
    a.seg = a.flux == 1 ? pick_seg(a.ny, a.nx, ctas * 4, C) : pick_seg(a.ny, a.nx, ctas * 4, C, 16, 64);
  a.seg = (a.seg + C - 1) / C * C;  // chunks never straddle segments
  a.nseg = (a.ny + a.seg - 1) / a.seg;
  a.band = pick_band(a.band, a.nx, a.nseg, ctas * 4, a.flux == 1 ? 2 : 3);
  const bool peer = a.halo_up || a.halo_dn;
  if (a.flux == 1) {
    if (peer) launch_sweep(sweep_y_kernel<1, true>, ctas, kExYSmemBytes, s, a, maps.ey_load, maps.ey_store);
    else launch_sweep(sweep_y_kernel<1, false>, ctas, kExYSmemBytes, s, a, maps.ey_load, maps.ey_store);
  } else {
    // the maps whose box is this TU's chunk (the tolerance TU's 4-cell
    // chunks share the exact-10 sweep's maps)
    const bool wide = Staging<1>::C == maps.y_cols;
    if (!wide && Staging<1>::C != maps.ey_cols) {
      std::fprintf(stderr, "hydro_b200: no tensor map for %d-cell row chunks\n", Staging<1>::C);
      std::abort();
    }
    const CUtensorMap& ld = wide ? maps.y_load : maps.ey_load;
    const CUtensorMap& st = wide ? maps.y_store : maps.ey_store;
    if (peer) launch_sweep(sweep_y_kernel<0, true>, ctas, kYSmemBytes, s, a, ld, st);
    else launch_sweep(sweep_y_kernel<0, false>, ctas, kYSmemBytes, s, a, ld, st);
  }
}

void HB_SWEEP(launch_sweep_xy)(const SweepArgs& a0, const CUtensorMap& load, const CUtensorMap& store,
                                const Geometry& geo, cudaStream_t s) {
  SweepArgs a = a0;
  const int ctas = geo.sms * geo.ctas_xy_per_sm;
  const int nbands = (a.ny + kFW - 1) / kFW;
  // rows per work item: about 4 items per CTA (dynamic balance against the 6
  // halo rows and the ring fill every item pays: config 1 -16% vs 8 items),
  // 4-row chunks, 32..256 rows
  if (a.seg <= 0) {
    long long seg = (long long)a.nx * nbands / ((long long)ctas * 4);
    if (seg < 32) seg = 32;
    if (seg > 256) seg = 256;
    a.seg = (int)seg;
  }
  a.seg = (a.seg + 3) / 4 * 4;
  a.nseg = (a.nx + a.seg - 1) / a.seg;
  const bool peer = a.halo_up || a.halo_dn;
  if (a.flux == 1) {  // exact-10 (whole domains: the caller keeps slabs on the split sweeps)
    if (a.last_step) launch_sweep_block(sweep_xy_kernel<1, false, 1>, ctas, 256, kFSmemBytesEx, s, a, load, store);
    else launch_sweep_block(sweep_xy_kernel<0, false, 1>, ctas, 256, kFSmemBytesEx, s, a, load, store);
  } else if (a.last_step) {
    if (peer) launch_sweep_block(sweep_xy_kernel<1, true, 0>, ctas, 256, kFSmemBytes, s, a, load, store);
    else launch_sweep_block(sweep_xy_kernel<1, false, 0>, ctas, 256, kFSmemBytes, s, a, load, store);
  } else {
    if (peer) launch_sweep_block(sweep_xy_kernel<0, true, 0>, ctas, 256, kFSmemBytes, s, a, load, store);
    else launch_sweep_block(sweep_xy_kernel<0, false, 0>, ctas, 256, kFSmemBytes, s, a, load, store);
  }
}

void HB_SWEEP(launch_prologue)(const PrologueArgs& a, cudaStream_t s) {
  // each thread walks ~nx/128 rows of its column: few enough warps that the
  // per-warp atomicMin of the dt limit does not serialise on one address
  dim3 grid((a.ny + 255) / 256, a.nx < 128 ? a.nx : 128);
  HB_SWEEP(prologue_kernel)<<<grid, 256, 0, s>>>(a);
}

#ifndef HB_TOLERANCE

void launch_ghost_fix(double* b, size_t pitch, int nx, int ny, int bc, cudaStream_t s) {
  if (bc != 0 || (ny & 31) != 1 || ny < 33) return;
  ghost_fix_kernel<<<(nx + 255) / 256, 256, 0, s>>>(b, pitch, nx, ny);
}

void launch_ghost_row_fix(double* a, size_t pitch, int nx, int ny, int bc, int wall_hi,
                          cudaStream_t s) {
  if (bc != 0 || !wall_hi || (nx & 31) != 1 || nx < 33) return;
  ghost_row_fix_kernel<<<(ny + 255) / 256, 256, 0, s>>>(a, pitch, nx, ny);
}

void launch_rows_to_tiles(const double* rows, size_t row_stride, double* u, size_t pitch, int v,
                          int i0, int n, int ny, cudaStream_t s) {
  dim3 grid((ny + 4 + 255) / 256, n < 1024 ? n : 1024);
  rows_tiles_kernel<<<grid, 256, 0, s>>>(const_cast<double*>(rows), row_stride, u, pitch, v, i0, n,
                                         ny, 1);
}

void launch_tiles_to_rows(const double* u, size_t pitch, double* rows, size_t row_stride, int v,
                          int i0, int n, int ny, cudaStream_t s) {
  dim3 grid((ny + 4 + 255) / 256, n < 1024 ? n : 1024);
  rows_tiles_kernel<<<grid, 256, 0, s>>>(rows, row_stride, const_cast<double*>(u), pitch, v, i0, n,
                                         ny, 0);
}

void launch_compare(const double* a, const double* b, size_t pitch, int nx, int ny,
                    unsigned long long* out, cudaStream_t s) {
  compare_kernel<<<1184, 256, 0, s>>>(a, b, pitch, nx, ny, out);
}

void launch_finish(const FinishArgs& a, cudaStream_t s) {
  const int n = a.nx + a.ny;
  finish_kernel<<<(n + 255) / 256, 256, 0, s>>>(a);
}

void launch_init(const InitArgs& a, cudaStream_t s) {
  dim3 grid((a.ny + 255) / 256, a.nx < 4096 ? a.nx : 4096);
  init_kernel<<<grid, 256, 0, s>>>(a);
}

void launch_row_audit(const double* u, size_t pitch, int nx, int ny, unsigned long long* hashes,
                      double* sums, cudaStream_t s) {
  const int n = 4 * nx;
  row_audit_kernel<<<(n + 127) / 128, 128, 0, s>>>(u, pitch, nx, ny, hashes, sums);
}

void launch_math_selftest(int op, const double* a, const double* b, double* fast, double* ref,
                          int* ok, size_t n, cudaStream_t s) {
  math_selftest_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(op, a, b, fast, ref, ok, n);
}

#endif  // !HB_TOLERANCE

}  // namespace hb
