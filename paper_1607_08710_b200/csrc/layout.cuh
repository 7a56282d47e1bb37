// layout.cuh -- device storage of a conserved field (4 fp64 SoA components).
//
// The reference stores each component as one ghosted row-major array of
// (nx+2gx) x (ny+2gy) doubles (grid.hpp:73-92, idx = j*nxt + i).  On the GPU a
// component is a pitched array with NG = 4 ghost layers on every side (the
// fused step reads a 4-wide halo of U^n) and its interior column 0 on a 128 B
// boundary, so every interior row is a coalesced, TMA-/vector-friendly run:
//
//   row j in [-NG, ny+NG), column i in [-NG, nx+NG)
//   at(c, i, j) = base + c*fstride + j*pitch + i
//   base        = alloc + NG*pitch + XPAD        (XPAD = 16 doubles = 128 B)
//
// pitch and fstride are multiples of 16 doubles.  A y-slab of a decomposed grid
// uses the same layout with ny = its local row count; its y ghost rows hold the
// neighbours' halo rows.
#pragma once

#include <cuda_runtime.h>  // __host__ / __device__ for host-only translation units too

#include <cstdint>

namespace lfb {

constexpr int NG = 4;       // device ghost layers (reference uses 2; the fused step needs 4)
constexpr int XPAD = 16;    // doubles from the allocation row start to interior column 0

struct Layout {
  int nx = 0, ny = 0;        // local interior extent
  int64_t pitch = 0;         // doubles per row
  int64_t fstride = 0;       // doubles per component
  int64_t alloc = 0;         // doubles per field allocation (4 components)

  static Layout make(int nx, int ny) {
    Layout L;
    L.nx = nx;
    L.ny = ny;
    L.pitch = ((int64_t)XPAD + nx + NG + 15) / 16 * 16;
    L.fstride = L.pitch * (int64_t)(ny + 2 * NG);
    // one spare row: the fused step's row copies of the last column strip may
    // run past the end of a row (the values are never used)
    L.alloc = 4 * L.fstride + (L.pitch > 256 ? L.pitch : 256);
    return L;
  }
  __host__ __device__ int64_t origin() const { return (int64_t)NG * pitch + XPAD; }
  __host__ __device__ int64_t off(int i, int j) const { return (int64_t)j * pitch + i; }
};

// The ghost fill (grid.cpp:72-114) as an index map: ghost layer l of a side of n
// cells reads cell src of the same row / column (n >= l: every source is interior);
// flip: a reflective image, times -1 in the normal momentum.  A corner is the y image
// of the x image (k_fill_xy's composition; multiplying by -1 is exact, so the order
// of the two does not matter).  bc: 0 transmissive, 1 reflective, 2 periodic.
__host__ __device__ inline int ghost_src(int i, int n, int lo, int hi, bool& flip) {
  flip = false;
  if (i < 0) {
    const int l = -i;
    if (lo == 0) return 0;
    if (lo == 1) {
      flip = true;
      return l - 1;
    }
    return n - l;
  }
  if (i >= n) {
    const int l = i - n + 1;
    if (hi == 0) return n - 1;
    if (hi == 1) {
      flip = true;
      return n - l;
    }
    return l - 1;
  }
  return i;
}

// A field: pointer to (component 0, i = 0, j = 0) plus the layout strides.
struct Field {
  double* p;
  int64_t pitch;
  int64_t fstride;
  __device__ __forceinline__ double& at(int c, int i, int j) const {
    return p[c * fstride + (int64_t)j * pitch + i];
  }
  __device__ __forceinline__ double* comp(int c) const { return p + c * fstride; }
};

}  // namespace lfb
