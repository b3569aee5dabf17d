// Compile-time lattice descriptors for the two coupled models the reference
// builds (config.cpp:404-410): D2Q9 flow + D2Q9 temperature (M = 18) and
// D3Q19 flow + D3Q7 temperature (M = 26). Plane order, opposites and weights
// are the reference's exactly (lattice.cpp:83-136); the coupled plane table
// is System::finalize's (collision.cpp:92-101): flow planes 0..MF-1, then the
// thermal planes. Everything is constexpr so the node kernels unroll to
// straight-line code with the velocity components folded in.
#pragma once
#include <cstdint>

namespace lbgpu {

struct LatD2 {
  static constexpr int DIM = 2, MF = 9, MT = 9, M = 18;
  static constexpr int NSHEAR = 2;
  __host__ __device__ static constexpr int ef(int j, int a) {
    constexpr int t[9][3] = {{0, 0, 0}, {1, 0, 0},  {-1, 0, 0}, {0, 1, 0},  {0, -1, 0},
                             {1, 1, 0}, {-1, 1, 0}, {1, -1, 0}, {-1, -1, 0}};
    return t[j][a];
  }
  __host__ __device__ static constexpr int et(int j, int a) { return ef(j, a); }
  __host__ __device__ static constexpr int oppf(int j) {
    constexpr int t[9] = {0, 2, 1, 4, 3, 8, 7, 6, 5};
    return t[j];
  }
  __host__ __device__ static constexpr int oppt(int j) { return oppf(j); }
  __host__ __device__ static constexpr double wf(int j) {
    return j == 0 ? 4.0 / 9 : (j <= 4 ? 1.0 / 9 : 1.0 / 36);
  }
  __host__ __device__ static constexpr double wt(int j) { return wf(j); }
  // MRT moment rows (lattice.cpp:31-50) evaluated at velocity j.
  __host__ __device__ static constexpr double U(int i, int j) {
    const double ex = ef(j, 0), ey = ef(j, 1);
    const double n2 = ex * ex + ey * ey;
    switch (i) {
      case 0: return 1.0;
      case 1: return 3.0 * n2 - 4.0;
      case 2: return 4.0 - 10.5 * n2 + 4.5 * n2 * n2;
      case 3: return ex;
      case 4: return (3.0 * n2 - 5.0) * ex;
      case 5: return ey;
      case 6: return (3.0 * n2 - 5.0) * ey;
      case 7: return ex * ex - ey * ey;
      default: return ex * ey;
    }
  }
  // Row classes of classify_rows (collision.cpp:31-44): 0 conserved, 1 shear, 2 other.
  __host__ __device__ static constexpr int row_class(int i) {
    return (i == 0 || i == 3 || i == 5) ? 0 : ((i == 7 || i == 8) ? 1 : 2);
  }
};

struct LatD3 {
  static constexpr int DIM = 3, MF = 19, MT = 7, M = 26;
  static constexpr int NSHEAR = 5;
  __host__ __device__ static constexpr int ef(int j, int a) {
    constexpr int t[19][3] = {{0, 0, 0},  {1, 0, 0},  {-1, 0, 0},  {0, 1, 0},  {0, -1, 0},
                              {0, 0, 1},  {0, 0, -1}, {1, 1, 0},   {-1, 1, 0}, {1, -1, 0},
                              {-1, -1, 0}, {1, 0, 1}, {-1, 0, 1},  {1, 0, -1}, {-1, 0, -1},
                              {0, 1, 1},  {0, -1, 1}, {0, 1, -1},  {0, -1, -1}};
    return t[j][a];
  }
  __host__ __device__ static constexpr int et(int j, int a) { return ef(j, a); }  // D3Q7 = first 7
  __host__ __device__ static constexpr int oppf(int j) {
    constexpr int t[19] = {0, 2, 1, 4, 3, 6, 5, 10, 9, 8, 7, 14, 13, 12, 11, 18, 17, 16, 15};
    return t[j];
  }
  __host__ __device__ static constexpr int oppt(int j) { return oppf(j); }
  __host__ __device__ static constexpr double wf(int j) {
    return j == 0 ? 1.0 / 3 : (j <= 6 ? 1.0 / 18 : 1.0 / 36);
  }
  __host__ __device__ static constexpr double wt(int j) { return j == 0 ? 0.0 : 1.0 / 6; }
  // MRT moment rows (lattice.cpp:52-81).
  __host__ __device__ static constexpr double U(int i, int j) {
    const double ex = ef(j, 0), ey = ef(j, 1), ez = ef(j, 2);
    const double n2 = ex * ex + ey * ey + ez * ez;
    switch (i) {
      case 0: return 1.0;
      case 1: return 19.0 * n2 - 30.0;
      case 2: return (21.0 * n2 * n2 - 53.0 * n2 + 24.0) / 2;
      case 3: return ex;
      case 4: return (5.0 * n2 - 9.0) * ex;
      case 5: return ey;
      case 6: return (5.0 * n2 - 9.0) * ey;
      case 7: return ez;
      case 8: return (5.0 * n2 - 9.0) * ez;
      case 9: return 3.0 * ex * ex - n2;
      case 10: return (3.0 * n2 - 5.0) * (3.0 * ex * ex - n2);
      case 11: return ey * ey - ez * ez;
      case 12: return (3.0 * n2 - 5.0) * (ey * ey - ez * ez);
      case 13: return ex * ey;
      case 14: return ey * ez;
      case 15: return ex * ez;
      case 16: return ex * (ey * ey - ez * ez);
      case 17: return ey * (ez * ez - ex * ex);
      default: return ez * (ex * ex - ey * ey);
    }
  }
  __host__ __device__ static constexpr int row_class(int i) {
    return (i == 0 || i == 3 || i == 5 || i == 7)
               ? 0
               : ((i == 9 || i == 11 || i == 13 || i == 14 || i == 15) ? 1 : 2);
  }
};

// Coupled plane helpers: p < MF is flow slot p, else thermal slot p - MF.
template <class L>
__host__ __device__ constexpr int cvel(int p, int a) {
  return p < L::MF ? L::ef(p, a) : L::et(p - L::MF, a);
}
template <class L>
__host__ __device__ constexpr int copp(int p) {
  return p < L::MF ? L::oppf(p) : L::MF + L::oppt(p - L::MF);
}

// Node code byte (one per node): tag in bits 0-2 (NodeTag order,
// collision.hpp:21), then flags.
enum : uint8_t {
  TAG_INTERIOR = 0, TAG_WALL = 1, TAG_INLET = 2, TAG_OUTLET = 3, TAG_HEATER = 4,
  TAG_MASK = 7,
  CODE_HAS_W = 8,      // w != 1 or design node: the node reads its design value
  CODE_SUPPORT = 16,   // objective support node (ObjectiveSpec::on_support)
  CODE_AXIS_SHIFT = 5, // bits 5-6: pressure-face normal axis
  CODE_NEG = 128,      // pressure-face normal sign is -1
  // An Interior node has no face normal: axis bits 11 mark an interior
  // design node (DesignField mask), for the one-shot update fused into the
  // next primal sweep.
  CODE_AXIS_BITS = 96,
  CODE_DESIGN_INT = 96,
};

}  // namespace lbgpu
