/*
 * hydro_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference hydro2d time step (the CPU results
 * oracle).  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * leg may load it, and only as the checker.  The product path
 * (paper_2106_13465_b200/, libhydro_b200.so) never links or calls it.
 *
 * Parity pin: the oracle reproduces the reference's own published digests
 * (proj/README.md:98-109) and is cross-checked against the unmodified
 * reference compiled from /root/reference (oracle/_ref, see oracle/Makefile).
 *
 * Storage: one contiguous buffer of 4 planes (rho, mom_x, mom_y, ener), each
 * (nx+4) x (ny+4) doubles, row-major with j fastest, plane v at offset
 * v*(nx+4)*(ny+4) -- the Grid2D layout of proj/include/hydro/grid.hpp:15-19,54-57.
 */
#ifndef HYDRO_ORACLE_H
#define HYDRO_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Boundary kinds.  REFLECT is the reference's only BC (grid.cpp:23-60);
 * TRANSMIT (zero-gradient: both ghost layers copy the adjacent interior
 * cell) is the BASELINE configs' extension. */
enum { OR_BC_REFLECT = 0, OR_BC_TRANSMIT = 1 };

/* Wall mask for slab runs: which ghost bands apply_boundary fills. */
enum { OR_WALL_XLO = 1, OR_WALL_XHI = 2, OR_WALL_Y = 4, OR_WALL_ALL = 7 };

/* Error categories, numbered like hydro::ErrorCategory + 1
 * (proj/include/hydro/errors.hpp:10-18); 0 = ok. */
enum {
  OR_OK = 0, OR_ERR_CONFIG = 1, OR_ERR_POSITIVITY = 2, OR_ERR_PROTOCOL = 3,
  OR_ERR_TASKGRAPH = 4, OR_ERR_EQUIVALENCE = 5, OR_ERR_IO = 6,
  OR_ERR_VALIDATION = 7
};

/* Error location: phase 0 = compute_dt, 1 = column sweep, 2 = row sweep;
 * loop 0 = primitive conversion (euler_kernel.cpp:124-139), 1 = Riemann
 * problem, 2 = conservative update (euler_kernel.cpp:200-220); field 0 = rho,
 * 1 = pres, 2 = internal energy, 3 = vacuum (exact-10 mode). */
typedef struct {
  int category;
  int step;
  int phase;
  int strip;
  int loop;
  int cell; /* strip-local index k - kGhost, as the reference prints it */
  int field;
  char message[256];
} oracle_error;

/* Case ids. */
enum {
  OR_CASE_UNIFORM = 0,      /* cases.cpp:11-21 with (1,0,0,1) as bench.cpp:32 */
  OR_CASE_BLAST = 1,        /* centred point explosion, cases.cpp:34-52 */
  OR_CASE_SOD_J = 2,        /* 4-row tube along j, cases.cpp:54-69 */
  OR_CASE_CORNER_BLAST = 3, /* BASELINE configs 0 and 3 */
  OR_CASE_SOD_X = 4,        /* BASELINE config 1 */
  OR_CASE_RANDOM = 5        /* BASELINE configs 2 and 4 */
};

size_t oracle_grid_doubles(int nx, int ny);

/* Fills u (zeroed first, like Grid2D's constructor) and the spacings. */
int oracle_init_case(double* u, int nx, int ny, int case_id, double gamma,
                     uint64_t seed, double* dx, double* dy, oracle_error* err);

/* Random-field initialiser restricted to global rows [row0, row0+nx) of a
 * (global_nx x ny) grid -- used to build slabs identical to the full grid. */
int oracle_init_random_rows(double* u, int nx, int ny, int row0, int global_nx,
                            double gamma, uint64_t seed, oracle_error* err);

void oracle_apply_boundary(double* u, int nx, int ny, int bc, int wall_mask);

/* min over interior cells of cell_dt_limit (before the cfl factor). */
int oracle_compute_limit(const double* u, int nx, int ny, double dx, double dy,
                         double gamma, double* limit, oracle_error* err);

/* One sweep over every strip of an axis (0 = Column, 1 = Row) with the given
 * dt, reading ghosts as they are.  step is only used for error context. */
int oracle_sweep_axis(double* u, int nx, int ny, double dx, double dy,
                      double gamma, int axis, double dt, oracle_error* err);

/* run_sequential (schedulers.cpp:103-116) with a BC kind. */
int oracle_run_sequential(double* u, int nx, int ny, double dx, double dy,
                          double gamma, double cfl, int bc, int steps,
                          double* last_dt, oracle_error* err);

/* advance_sequential (schedulers.cpp:95-101). */
int oracle_advance(double* u, int nx, int ny, double dx, double dy,
                   double gamma, int bc, double dt, oracle_error* err);

/* run_until (schedulers.cpp:118-138). */
int oracle_run_until(double* u, int nx, int ny, double dx, double dy,
                     double gamma, double cfl, int bc, double t_end,
                     int* steps, oracle_error* err);

/* sweep_strip on an AoS strip of n+4 cells {rho, mom_a, mom_b, ener}
 * (euler_kernel.cpp:111-223).  first/last receive the boundary fluxes. */
int oracle_sweep_strip(double* cells, int n, double dx, double dt, double gamma,
                       double* first, double* last, oracle_error* err);

/* Interface flux used by every sweep: 0 = HLLC (default, the reference hot
 * path), 1 = exact-10 (exact Riemann solver, 10 Newton iterations). */
void oracle_set_flux(int flux);
/* Strip-parallel sweeps with n threads (long golden runs; see hydro_oracle.c). */
void oracle_set_threads(int n);
int oracle_exact10_flux(const double* wl, const double* wr, double gamma, double* flux);

/* riemann_flux (euler_kernel.cpp:59-109) on primitive states. */
int oracle_riemann_flux(const double* wl, const double* wr, double gamma,
                        double* flux, oracle_error* err);

/* Audit (audit.cpp:16-76, 137-154). */
uint64_t oracle_digest(const double* u, int nx, int ny);
void oracle_sums(const double* u, int nx, int ny, double sums[4]);
void oracle_compare_tolerance(const double* a, const double* b, int nx, int ny,
                              double* max_rel, double* l1_rel);

uint64_t oracle_splitmix64(uint64_t x);

#ifdef __cplusplus
}
#endif

#endif
