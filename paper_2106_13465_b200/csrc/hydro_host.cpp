// hydro_host.cpp -- host utilities of libhydro_b200.so (no device needed).
//
//  * hydro_grid_digest: the reference's FNV-1a digest over the interior
//    bytes, plane by plane, i then j (proj/src/audit.cpp:53-76), used as the
//    bitwise equivalence gate between this library and the reference.
//  * hydro_init_case_host: the reference's initial conditions
//    (proj/src/cases.cpp:11-69) plus the BASELINE configs' corner blast,
//    planar Sod along i and seeded random field; bitwise equal to the device
//    initialiser (init_kernel in hydro_kernels.cu).
// Built with -ffp-contract=off like the reference (proj/CMakeLists.txt:10-14).
#include <cstdint>
#include <cstring>
#include <vector>

#include "../../include/hydro_gpu.h"

namespace {

struct P { double r, va, vb, p; };

uint64_t mix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

double sym_unit(uint64_t seed, uint64_t cell, int var) {
  const uint64_t h = mix64(seed ^ (4ull * cell + (uint64_t)var));
  return 2.0 * ((double)(h >> 11) * 0x1.0p-53) - 1.0;
}

void put(double* const planes[4], size_t stride, int i, int j, const P& w, double gamma) {
  // prim_to_cons, euler_kernel.cpp:22-28
  const size_t at = (size_t)(i + 1) * stride + (size_t)(j + 1);
  planes[0][at] = w.r;
  planes[1][at] = w.r * w.va;
  planes[2][at] = w.r * w.vb;
  planes[3][at] = w.p / (gamma - 1.0) + 0.5 * w.r * (w.va * w.va + w.vb * w.vb);
}

}  // namespace

extern "C" {

uint64_t hydro_grid_digest(const double* const planes[4], size_t stride, int nx, int ny) {
  uint64_t h = 14695981039346656037ull;
  for (int v = 0; v < 4; ++v) {
    for (int i = 1; i <= nx; ++i) {
      const double* row = planes[v] + (size_t)(i + 1) * stride + 2;
      for (int j = 0; j < ny; ++j) {
        uint64_t bits;
        std::memcpy(&bits, row + j, 8);
        for (int b = 0; b < 8; ++b) {
          h ^= (bits >> (8 * b)) & 0xffu;
          h *= 1099511628211ull;
        }
      }
    }
  }
  return h;
}

uint64_t hydro_fnv1a_rows(uint64_t h, const double* plane, size_t stride, int nx, int ny) {
  for (int i = 1; i <= nx; ++i) {
    const double* row = plane + (size_t)(i + 1) * stride + 2;
    for (int j = 0; j < ny; ++j) {
      uint64_t bits;
      std::memcpy(&bits, row + j, 8);
      for (int b = 0; b < 8; ++b) {
        h ^= (bits >> (8 * b)) & 0xffu;
        h *= 1099511628211ull;
      }
    }
  }
  return h;
}

uint64_t hydro_combine_row_hashes(const uint64_t* row_hashes, size_t n) {
  uint64_t h = 14695981039346656037ull;
  for (size_t k = 0; k < n; ++k)
    for (int b = 0; b < 8; ++b) {
      h ^= (row_hashes[k] >> (8 * b)) & 0xffu;
      h *= 1099511628211ull;
    }
  return h;
}

uint64_t hydro_grid_state_hash(const double* const planes[4], size_t stride, int nx, int ny) {
  std::vector<uint64_t> rows(4 * (size_t)nx);
  for (int v = 0; v < 4; ++v)
    for (int i = 1; i <= nx; ++i) {
      const double* row = planes[v] + (size_t)(i + 1) * stride + 2;
      uint64_t h = 14695981039346656037ull;
      for (int j = 0; j < ny; ++j) {
        uint64_t bits;
        std::memcpy(&bits, row + j, 8);
        for (int b = 0; b < 8; ++b) {
          h ^= (bits >> (8 * b)) & 0xffu;
          h *= 1099511628211ull;
        }
      }
      rows[(size_t)v * nx + (i - 1)] = h;
    }
  return hydro_combine_row_hashes(rows.data(), rows.size());
}

// pairwise_sum (audit.cpp:16-25): halve until blocks of <= 8.
double hydro_pairwise_sum(const double* v, size_t n) {
  if (n <= 8) {
    double s = 0.0;
    for (size_t k = 0; k < n; ++k) s += v[k];
    return s;
  }
  const size_t h = n / 2;
  return hydro_pairwise_sum(v, h) + hydro_pairwise_sum(v + h, n - h);
}

int hydro_init_case_host(int case_id, int nx, int ny, double gamma, uint64_t seed,
                         double* const planes[4], size_t stride, double* dx, double* dy) {
  if (nx < 4 || ny < 4 || stride < (size_t)ny + 4) return HYDRO_GPU_ERR_CONFIG;
  if (case_id == HYDRO_GPU_CASE_SOD_J && (nx != 4 || ny < 8)) return HYDRO_GPU_ERR_CONFIG;
  if (case_id < 0 || case_id > 5) return HYDRO_GPU_ERR_CONFIG;
  for (int v = 0; v < 4; ++v) std::memset(planes[v], 0, sizeof(double) * (size_t)(nx + 4) * stride);
  double hx = 1.0 / nx, hy = 1.0 / ny;
  if (case_id == HYDRO_GPU_CASE_SOD_J) hx = hy = 1.0 / ny;
  if (dx) *dx = hx;
  if (dy) *dy = hy;
  const P left = {1.0, 0.0, 0.0, 1.0}, right = {0.125, 0.0, 0.0, 0.1};
  for (int i = 1; i <= nx; ++i) {
    for (int j = 1; j <= ny; ++j) {
      P w = {1.0, 0.0, 0.0, 1.0};
      switch (case_id) {
        case HYDRO_GPU_CASE_BLAST: w.p = 1e-5 * (gamma - 1.0); break;
        case HYDRO_GPU_CASE_CORNER_BLAST: w.p = 1e-5; break;
        case HYDRO_GPU_CASE_SOD_J: w = (j <= ny / 2) ? left : right; break;
        case HYDRO_GPU_CASE_SOD_X: w = (i <= nx / 2) ? left : right; break;
        case HYDRO_GPU_CASE_RANDOM: {
          const uint64_t cell = (uint64_t)(i - 1) * (uint64_t)ny + (uint64_t)(j - 1);
          w.r = 1.0 + 0.1 * sym_unit(seed, cell, 0);
          w.p = 1.0 + 0.1 * sym_unit(seed, cell, 1);
          w.va = 0.1 * sym_unit(seed, cell, 2);
          w.vb = 0.1 * sym_unit(seed, cell, 3);
          break;
        }
        default: break;
      }
      put(planes, stride, i, j, w, gamma);
    }
  }
  if (case_id == HYDRO_GPU_CASE_BLAST) {  // cases.cpp:34-52
    const int ni = nx % 2 ? 1 : 2, nj = ny % 2 ? 1 : 2;
    const int i0 = nx % 2 ? (nx + 1) / 2 : nx / 2, j0 = ny % 2 ? (ny + 1) / 2 : ny / 2;
    const double share = 1.0 / ((double)ni * (double)nj);
    for (int a = 0; a < ni; ++a)
      for (int b = 0; b < nj; ++b)
        planes[3][(size_t)(i0 + a + 1) * stride + (size_t)(j0 + b + 1)] = share / (hx * hy);
  }
  if (case_id == HYDRO_GPU_CASE_CORNER_BLAST)
    planes[3][(size_t)2 * stride + 2] = 1.0 / (hx * hy);
  return HYDRO_GPU_OK;
}

}  // extern "C"
