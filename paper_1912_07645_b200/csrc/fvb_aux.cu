// Auxiliary kernels of the hot path (mode-independent, compiled -fmad=false):
//   * ghost fill on padded buffers (grid.py:147-175 fill_axis / fill_boundary)
//   * halo slab pack/unpack for the NCCL exchange (parallel.py:185-254)
//   * per-sample Welford/Chan moment merge (uq.py:114-158)
//   * structure-function sums (uq.py:231-273), deterministic two-pass reduce
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "../../include/fvb200.h"
#include "fvb_state.cuh"

namespace fvb {

__global__ void export_kernel(const FvbState* st, int dim, double* out) { export_step(st, dim, out); }
__global__ void finalize_global_kernel(FvbState* st, LoopCtl L, const double* g, int post) {
  finalize_global(st, L, g, post != 0);
}
int launch_export(const FvbState* st, int dim, double* out, cudaStream_t s) {
  export_kernel<<<1, 1, 0, s>>>(st, dim, out);
  return 0;
}
int launch_finalize_global(FvbState* st, const LoopCtl& L, const double* g, int post, cudaStream_t s) {
  finalize_global_kernel<<<1, 1, 0, s>>>(st, L, g, post);
  return 0;
}

namespace {

struct Pad {
  int64_t P[3];   // padded extents (x first); unused axes 1
  int64_t n[3];   // interior extents
  int g;
  int dim;
};

__host__ __device__ inline Pad make_pad(const fvb_scheme& s) {
  Pad p;
  p.g = s.ghost;
  p.dim = s.dim;
  for (int k = 0; k < 3; ++k) {
    p.n[k] = k < s.dim ? s.cells[k] : 1;
    p.P[k] = k < s.dim ? s.cells[k] + 2 * s.ghost : 1;
  }
  return p;
}

// padded coordinate -> element offset relative to the interior origin
__device__ inline int64_t poff(const Pad& p, const fvb_layout& L, int64_t px, int64_t py, int64_t pz) {
  int64_t o = px - (p.dim >= 1 ? p.g : 0);
  if (p.dim >= 2) o += (py - p.g) * L.sy;
  if (p.dim >= 3) o += (pz - p.g) * L.sz;
  return o;
}

// fill_axis: both ghost slabs of one axis, full padded extent of the others
__global__ void fill_axis_kernel(Pad p, fvb_layout L, double* u, int ncomp, int ninst, int axis, int periodic) {
  int64_t E[3] = {p.P[0], p.P[1], p.P[2]};
  E[axis] = 2 * p.g;
  const int64_t per = E[0] * E[1] * E[2];
  const int64_t total = per * ncomp * ninst;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i;
    int64_t c3[3];
    c3[0] = r % E[0]; r /= E[0];
    c3[1] = r % E[1]; r /= E[1];
    c3[2] = r % E[2]; r /= E[2];
    const int c = (int)(r % ncomp);
    const int inst = (int)(r / ncomp);
    const int64_t j = c3[axis];
    const int64_t n = p.n[axis];
    int64_t dst, src;
    if (j < p.g) {               // low ghosts [0, g)
      dst = j;
      src = periodic ? n + j : p.g;
    } else {                     // high ghosts [n+g, n+2g)
      dst = n + j;
      src = periodic ? j : n + p.g - 1;
    }
    int64_t d3[3] = {c3[0], c3[1], c3[2]};
    int64_t s3[3] = {c3[0], c3[1], c3[2]};
    d3[axis] = dst;
    s3[axis] = src;
    double* b = u + L.origin + inst * L.si + c * L.sc;
    b[poff(p, L, d3[0], d3[1], d3[2])] = b[poff(p, L, s3[0], s3[1], s3[2])];
  }
}

// halo slab: side 0 = low face, side 1 = high face.
// pack reads the g interior layers next to the face, unpack writes the ghosts.
__global__ void halo_kernel(Pad p, fvb_layout L, double* u, int ncomp, int axis, int side, double* buf,
                            int unpack) {
  int64_t E[3] = {p.P[0], p.P[1], p.P[2]};
  E[axis] = p.g;
  const int64_t total = E[0] * E[1] * E[2] * ncomp;
  const int64_t n = p.n[axis];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i;
    int64_t c3[3];
    c3[0] = r % E[0]; r /= E[0];
    c3[1] = r % E[1]; r /= E[1];
    c3[2] = r % E[2]; r /= E[2];
    const int c = (int)r;
    const int64_t j = c3[axis];
    int64_t a;
    if (unpack) a = side == 0 ? j : n + p.g + j;  // ghosts
    else a = side == 0 ? p.g + j : n + j;         // parallel.py:237-239
    c3[axis] = a;
    double* b = u + L.origin + c * L.sc;
    const int64_t o = poff(p, L, c3[0], c3[1], c3[2]);
    if (unpack) b[o] = buf[i];
    else buf[i] = b[o];
  }
}

// Samples inst .. inst+nbatch-1 merged, in that order, into (mean, m2)
// holding `count` samples.  Each sample is a fresh MomentAccumulator after
// update(v) (uq.py:125-133 with count 0):
//   om = 0 + (v - 0)/1,  om2 = 0 + (v - 0)*(v - om)
// merged by uq.py:135-148 (the first merge copies).  The running (mean, m2)
// of an element stay in registers across the batch: the statistics cost
// one read + one write of (mean, m2) per BATCH instead of per sample, with
// the exact operation sequence of nbatch single merges (bitwise equal).
constexpr int kMomMaxBatch = 64;

__global__ void moments_push_kernel(Pad p, fvb_layout L, const double* u, int ncomp, int inst, int nbatch,
                                    double* mean, double* m2, long long count) {
  __shared__ double fracs[kMomMaxBatch];  // other.count / total (int / int) of merge b
  for (int b = threadIdx.x; b < nbatch; b += blockDim.x) fracs[b] = 1.0 / (double)(count + b + 1);
  __syncthreads();
  // block-strided over (component, z, y) rows, threads over x: no per-element
  // index division; the (mean, m2) arrays are dense (ncomp, z, y, x)
  const int64_t nrow = p.n[1] * p.n[2];
  for (int64_t row = blockIdx.x; row < nrow * ncomp; row += gridDim.x) {
    const int c = (int)(row / nrow);
    const int64_t yz = row - (int64_t)c * nrow;
    const int64_t y = yz % p.n[1], z = yz / p.n[1];
    const double* src = u + L.origin + inst * L.si + c * L.sc + y * L.sy + z * L.sz;
    double* mrow = mean + row * p.n[0];
    double* qrow = m2 + row * p.n[0];
    for (int64_t x = threadIdx.x; x < p.n[0]; x += blockDim.x) {
      double mu = 0.0, q = 0.0;
      if (count > 0) {
        mu = mrow[x];
        q = qrow[x];
      }
      for (int b = 0; b < nbatch; ++b) {
        const double v = src[b * L.si + x];
        const double d0 = v - 0.0;
        const double om = 0.0 + d0 / 1.0;
        const double om2 = 0.0 + d0 * (v - om);
        if (count + b == 0) {
          mu = om;
          q = om2;
        } else {
          const double frac = fracs[b];
          const double fc = (double)(count + b);
          const double delta = om - mu;
          mu = mu + delta * frac;
          q = (q + om2) + ((delta * delta) * fc) * frac;
        }
      }
      mrow[x] = mu;
      qrow[x] = q;
    }
  }
}

__global__ void moments_merge_kernel(double* ma, double* m2a, long long ca, const double* mb, const double* m2b,
                                     long long cb, int64_t n) {
  const double total = (double)(ca + cb);
  const double frac = (double)cb / total;
  const double fca = (double)ca;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (cb == 0) continue;
    if (ca == 0) {
      ma[i] = mb[i];
      m2a[i] = m2b[i];
      continue;
    }
    const double delta = mb[i] - ma[i];
    const double m = ma[i] + delta * frac;
    m2a[i] = (m2a[i] + m2b[i]) + ((delta * delta) * fca) * frac;
    ma[i] = m;
  }
}

constexpr int kSfThreads = 256;

// Pass 1: per-block partial sums S[h][j] of |w(x + h e_j) - w(x)|^p, where
// j is the NUMPY axis (0 = slowest), matching np.roll(w, -h, axis=j).
// Blocks stride over the (z, y) rows, threads over x (no per-element index
// division); the shifted reads hit L2 (the field is L2-resident).  Fixed
// partition and reduction order: deterministic.
__global__ void __launch_bounds__(kSfThreads) structure_pass1(Pad p, fvb_layout L, const double* u, int inst,
                                                              int comp, double pw, int H, double* partials) {
  __shared__ double red[kSfThreads / 32];
  const int dim = p.dim;
  const int64_t nrow = p.n[1] * p.n[2];
  const double* w = u + L.origin + inst * L.si + comp * L.sc;
  for (int h = 0; h <= H; ++h) {
    for (int j = 0; j < dim; ++j) {
      const int k = dim - 1 - j;  // spatial axis of numpy axis j
      const int64_t hk = h % p.n[k];
      double acc = 0.0;
      for (int64_t row = blockIdx.x; row < nrow; row += gridDim.x) {
        const int64_t y = row % p.n[1], z = row / p.n[1];
        const int64_t o = y * L.sy + z * L.sz;
        int64_t os = o;  // shifted row for k = 1, 2
        if (k == 1) os = ((y + hk < p.n[1]) ? y + hk : y + hk - p.n[1]) * L.sy + z * L.sz;
        if (k == 2) os = y * L.sy + ((z + hk < p.n[2]) ? z + hk : z + hk - p.n[2]) * L.sz;
        for (int64_t x = threadIdx.x; x < p.n[0]; x += blockDim.x) {
          const int64_t xs = k == 0 ? ((x + hk < p.n[0]) ? x + hk : x + hk - p.n[0]) : x;
          const double d = fabs(w[os + xs] - w[o + x]);
          acc += pw == 2.0 ? d * d : (pw == 1.0 ? d : pow(d, pw));
        }
      }
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
      if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
      __syncthreads();
      if (threadIdx.x == 0) {
        double s = 0.0;
        for (int q = 0; q < kSfThreads / 32; ++q) s += red[q];
        partials[((int64_t)blockIdx.x * (H + 1) + h) * dim + j] = s;
      }
      __syncthreads();
    }
  }
}

// Pass 2 (one block): fixed-order sum of the partials -- one warp per
// (offset h, numpy axis j) pair, lane-strided over the blocks then a
// shuffle tree -- and the reference's accumulation acc = sum_j mean_j ;
// sums[h] += acc / dim (uq.py:257-261).  Offsets go in chunks of 8, so any
// max offset works with a fixed-size table.
__global__ void structure_pass2(const double* __restrict__ partials, int nblocks, int H, int dim, double ncell,
                                double* sums) {
  __shared__ double S[8 * 3];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  for (int hb = 0; hb <= H; hb += 8) {
    for (int k = warp; k < 8 * dim; k += nwarps) {
      const int h = hb + k / dim, j = k % dim;
      if (h > H) continue;
      double acc = 0.0;
      for (int b = lane; b < nblocks; b += 32) acc += partials[((int64_t)b * (H + 1) + h) * dim + j];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
      if (lane == 0) S[k] = acc;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int h = hb; h <= H && h < hb + 8; ++h) {
        double accj = 0.0;
        for (int j = 0; j < dim; ++j) accj += S[(h - hb) * dim + j] / ncell;
        sums[h] += accj / dim;
      }
    }
    __syncthreads();
  }
}

// Face-only halo exchange between subdomain instances of one buffer
// (parallel.py:201-254 with the corner passes dropped: the residual crops
// transverse axes to the interior, solver.py:99-104, so corners are never
// read).  Instance i is rank i of a Cartesian topology, x fastest
// (parallel.py:66-77).  Ghosts on split axes come from the neighbour's
// interior (periodic wrap at the world edge) or, at a non-periodic world
// edge, from the nearest own interior cell (parallel.py:189-198).
struct Topo {
  int r[3];       // ranks per axis
  int periodic[3];
};

__global__ void halo_instances_kernel(Pad p, fvb_layout L, double* u, int ncomp, int ninst, Topo T) {
  const int64_t nx = p.n[0], ny = p.n[1], nz = p.n[2];
  const int g = p.g;
  int64_t per_axis[3];
  per_axis[0] = (T.r[0] > 1) ? 2LL * g * ny * nz : 0;
  per_axis[1] = (T.r[1] > 1) ? 2LL * g * nx * nz : 0;
  per_axis[2] = (T.r[2] > 1) ? 2LL * g * nx * ny : 0;
  const int64_t per_comp = per_axis[0] + per_axis[1] + per_axis[2];
  const int64_t total = per_comp * ncomp * ninst;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t q = i % per_comp;
    const int64_t cc = i / per_comp;
    const int c = (int)(cc % ncomp);
    const int inst = (int)(cc / ncomp);
    int axis = 0;
    while (q >= per_axis[axis]) { q -= per_axis[axis]; ++axis; }
    const int a1 = axis == 0 ? 1 : 0, a2 = axis == 2 ? 1 : 2;
    const int64_t t0 = q % p.n[a1];
    q /= p.n[a1];
    const int64_t t1 = q % p.n[a2];
    q /= p.n[a2];
    const int j = (int)(q % g);
    const int side = (int)(q / g);
    int nb[3] = {inst % T.r[0], (inst / T.r[0]) % T.r[1], inst / (T.r[0] * T.r[1])};
    const int64_t n = p.n[axis];
    int64_t src_a;
    int src_inst;
    nb[axis] += side == 0 ? -1 : 1;
    if ((nb[axis] < 0 || nb[axis] >= T.r[axis]) && !T.periodic[axis]) {
      src_inst = inst;                 // outflow world edge: nearest own interior cell
      src_a = side == 0 ? 0 : n - 1;
    } else {
      nb[axis] = (nb[axis] + T.r[axis]) % T.r[axis];
      src_inst = nb[0] + T.r[0] * (nb[1] + T.r[1] * nb[2]);
      src_a = side == 0 ? n - g + j : j;   // neighbour's interior slab
    }
    const int64_t dst_a = side == 0 ? (int64_t)j - g : n + j;
    int64_t d3[3], s3[3];
    d3[axis] = dst_a;
    s3[axis] = src_a;
    d3[a1] = s3[a1] = t0;
    d3[a2] = s3[a2] = t1;
    const int64_t od = d3[0] + (p.dim >= 2 ? d3[1] * L.sy : 0) + (p.dim >= 3 ? d3[2] * L.sz : 0);
    const int64_t os = s3[0] + (p.dim >= 2 ? s3[1] * L.sy : 0) + (p.dim >= 3 ? s3[2] * L.sz : 0);
    double* base = u + L.origin + c * L.sc;
    base[inst * L.si + od] = base[src_inst * L.si + os];
  }
}

// ---------------------------------------------------------------------------
// Device initial data: the reference's initial-data
// expression language (iodsl/expr.py:338-386 eval_init) compiled on the host
// into a stack bytecode (initdev.py) and evaluated per cell centre, for every
// sample of a batch, straight into the padded batch buffer.  IEEE + - * / and
// sqrt match numpy bitwise (this unit is built -fmad=false); sin / cos / exp
// / pow are CUDA's (<= 2 ulp), so the result is rounding-level close to the
// reference, not bitwise.
// ---------------------------------------------------------------------------
enum InitOp : int {
  IO_CONST = 0, IO_X, IO_Y, IO_Z, IO_RAND, IO_NEG, IO_ADD, IO_SUB, IO_MUL, IO_DIV, IO_POW, IO_LT, IO_LE, IO_GT,
  IO_GE, IO_EQ, IO_NE, IO_SEL, IO_SIN, IO_COS, IO_EXP, IO_ABS, IO_SQRT, IO_MIN, IO_MAX, IO_SQR, IO_RECIP
};
constexpr int kInitStack = 32;


__device__ __forceinline__ double np_maximum(double a, double b) { return (a > b || a != a) ? a : b; }
__device__ __forceinline__ double np_minimum(double a, double b) { return (a < b || a != a) ? a : b; }

__device__ double init_run(const InitArgs& A, int c, const double* X, double cx, double cy, double cz) {
  double st[kInitStack];
  int sp = 0;
  for (int i = A.off[c]; i < A.off[c + 1]; ++i) {
    const int w = A.code[i];
    const int op = w & 0xff, arg = w >> 8;
    switch (op) {
      case IO_CONST: st[sp++] = A.k[arg]; break;
      case IO_X: st[sp++] = cx; break;
      case IO_Y: st[sp++] = cy; break;
      case IO_Z: st[sp++] = cz; break;
      case IO_RAND: st[sp++] = X[arg]; break;
      case IO_NEG: st[sp - 1] = -st[sp - 1]; break;
      case IO_SIN: st[sp - 1] = sin(st[sp - 1]); break;
      case IO_COS: st[sp - 1] = cos(st[sp - 1]); break;
      case IO_EXP: st[sp - 1] = exp(st[sp - 1]); break;
      case IO_ABS: st[sp - 1] = fabs(st[sp - 1]); break;
      case IO_SQRT: st[sp - 1] = sqrt(st[sp - 1]); break;
      case IO_SQR: st[sp - 1] = st[sp - 1] * st[sp - 1]; break;
      case IO_RECIP: st[sp - 1] = 1.0 / st[sp - 1]; break;
      case IO_SEL: {  // cond ? a : b  (np.where(cond != 0, a, b))
        const double b = st[--sp], a = st[--sp], q = st[sp - 1];
        st[sp - 1] = q != 0.0 ? a : b;
        break;
      }
      default: {
        const double b = st[--sp], a = st[sp - 1];
        double r;
        switch (op) {
          case IO_ADD: r = a + b; break;
          case IO_SUB: r = a - b; break;
          case IO_MUL: r = a * b; break;
          case IO_DIV: r = a / b; break;
          case IO_POW: r = pow(a, b); break;
          case IO_LT: r = a < b ? 1.0 : 0.0; break;
          case IO_LE: r = a <= b ? 1.0 : 0.0; break;
          case IO_GT: r = a > b ? 1.0 : 0.0; break;
          case IO_GE: r = a >= b ? 1.0 : 0.0; break;
          case IO_EQ: r = a == b ? 1.0 : 0.0; break;
          case IO_NE: r = a != b ? 1.0 : 0.0; break;
          case IO_MIN: r = np_minimum(a, b); break;
          default: r = np_maximum(a, b); break;  // IO_MAX
        }
        st[sp - 1] = r;
      }
    }
  }
  return st[0];
}

// bad[inst * (ncomp + 2) + j]: lowest flat cell (numpy order) where
// component j is non-finite (j < ncomp), the primitive state is
// non-positive (j = ncomp), the conserved state is unphysical (ncomp + 1)
__global__ void init_eval_kernel(InitArgs A, fvb_layout L, const double* vecs, int ninst, double* out,
                                 unsigned long long* bad) {
  const int64_t ncell = A.n[0] * A.n[1] * A.n[2];
  const double floor_ = 1e-12;  // equations.py POSITIVITY_FLOOR
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ncell * ninst;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int inst = (int)(i / ncell);
    const int64_t cell = i - inst * ncell;
    const int64_t x = cell % A.n[0], y = (cell / A.n[0]) % A.n[1], z = cell / (A.n[0] * A.n[1]);
    // grid.py cell_centers: origin + (i + 0.5) * delta
    const double cx = A.origin[0] + ((double)x + 0.5) * A.delta[0];
    const double cy = A.dim >= 2 ? A.origin[1] + ((double)y + 0.5) * A.delta[1] : 0.0;
    const double cz = A.dim >= 3 ? A.origin[2] + ((double)z + 0.5) * A.delta[2] : 0.0;
    const double* X = vecs + (int64_t)inst * (A.nrand > 0 ? A.nrand : 1);
    unsigned long long* b = bad + (int64_t)inst * (A.ncomp + 2);
    double v[5];
    for (int c = 0; c < A.ncomp; ++c) {
      v[c] = init_run(A, c, X, cx, cy, cz);
      if (!isfinite(v[c])) atomicMin(&b[c], (unsigned long long)cell);
    }
    if (A.euler) {
      const int d = A.dim;
      if (A.primitive) {  // equations.py:132-145 primitive_to_conserved
        const double rho = v[0], p = v[1 + d];
        if (rho <= floor_ || p <= floor_) atomicMin(&b[A.ncomp], (unsigned long long)cell);
        double kin = 0.0;
        for (int k = 0; k < d; ++k) {
          kin = kin + v[1 + k] * v[1 + k];
          v[1 + k] = rho * v[1 + k];
        }
        v[1 + d] = p / (A.gamma - 1.0) + 0.5 * rho * kin;
      }
      // equations.py:62-73 pressure / physical_mask
      double msq = 0.0;
      for (int k = 0; k < d; ++k) msq = msq + v[1 + k] * v[1 + k];
      const double pr = (A.gamma - 1.0) * (v[1 + d] - msq / (2.0 * v[0]));
      if (!(v[0] > floor_ && pr > floor_)) atomicMin(&b[A.ncomp + 1], (unsigned long long)cell);
    }
    double* o = out + inst * L.si + L.origin + x + y * L.sy + z * L.sz;
    for (int c = 0; c < A.ncomp; ++c) o[c * L.sc] = v[c];
  }
}

int grid_for(int64_t n) {
  int64_t b = (n + 255) / 256;
  if (b > 148 * 16) b = 148 * 16;
  if (b < 1) b = 1;
  return (int)b;
}

}  // namespace

int launch_fill_axis(const fvb_scheme& s, const fvb_layout& L, double* u, int ninst, int axis, cudaStream_t st) {
  const Pad p = make_pad(s);
  int64_t n = (int64_t)2 * p.g * s.ncomp * ninst;
  for (int k = 0; k < 3; ++k)
    if (k != axis) n *= p.P[k];
  fill_axis_kernel<<<grid_for(n), 256, 0, st>>>(p, L, u, s.ncomp, ninst, axis, s.bc[axis] == FVB_BC_PERIODIC);
  return 0;
}

int64_t halo_count(const fvb_scheme& s, int axis) {
  const Pad p = make_pad(s);
  int64_t n = (int64_t)p.g * s.ncomp;
  for (int k = 0; k < 3; ++k)
    if (k != axis) n *= p.P[k];
  return n;
}

int launch_halo(const fvb_scheme& s, const fvb_layout& L, double* u, int axis, int side, double* buf, int unpack,
                cudaStream_t st) {
  const Pad p = make_pad(s);
  halo_kernel<<<grid_for(halo_count(s, axis)), 256, 0, st>>>(p, L, u, s.ncomp, axis, side, buf, unpack);
  return 0;
}

int launch_halo_instances(const fvb_scheme& s, const fvb_layout& L, double* u, int ninst, const int* ranks,
                          const int* periodic, cudaStream_t st) {
  const Pad p = make_pad(s);
  Topo T;
  int64_t per = 0;
  for (int k = 0; k < 3; ++k) {
    T.r[k] = k < s.dim ? ranks[k] : 1;
    T.periodic[k] = periodic[k];
  }
  if (T.r[0] > 1) per += 2LL * p.g * p.n[1] * p.n[2];
  if (T.r[1] > 1) per += 2LL * p.g * p.n[0] * p.n[2];
  if (T.r[2] > 1) per += 2LL * p.g * p.n[0] * p.n[1];
  if (per == 0) return 0;
  halo_instances_kernel<<<grid_for(per * s.ncomp * ninst), 256, 0, st>>>(p, L, u, s.ncomp, ninst, T);
  return 1;
}

int launch_moments_push(const fvb_scheme& s, const fvb_layout& L, const double* u, int inst, int nbatch, double* mean,
                        double* m2, int64_t count_before, cudaStream_t st) {
  const Pad p = make_pad(s);
  const int64_t rows = p.n[1] * p.n[2] * s.ncomp;
  const int blocks = (int)std::min<int64_t>(rows, 148 * 16);
  for (int b0 = 0; b0 < nbatch; b0 += kMomMaxBatch)
    moments_push_kernel<<<blocks, 256, 0, st>>>(p, L, u, s.ncomp, inst + b0, std::min(kMomMaxBatch, nbatch - b0), mean,
                                                m2, (long long)count_before + b0);
  return 0;
}

int launch_moments_merge(double* ma, double* m2a, int64_t ca, const double* mb, const double* m2b, int64_t cb,
                         int64_t n, cudaStream_t st) {
  moments_merge_kernel<<<grid_for(n), 256, 0, st>>>(ma, m2a, (long long)ca, mb, m2b, (long long)cb, n);
  return 0;
}

int structure_blocks(const fvb_scheme& s) {
  const Pad p = make_pad(s);
  const int64_t rows = p.n[1] * p.n[2];
  return (int)std::min<int64_t>(rows, 148 * 8);
}

int launch_structure(const fvb_scheme& s, const fvb_layout& L, const double* u, int inst, int comp, double pw,
                     int H, double* d_sums, double* d_partials, int nblocks, cudaStream_t st) {
  const Pad p = make_pad(s);
  structure_pass1<<<nblocks, kSfThreads, 0, st>>>(p, L, u, inst, comp, pw, H, d_partials);
  structure_pass2<<<1, kSfThreads, 0, st>>>(d_partials, nblocks, H, s.dim, (double)(p.n[0] * p.n[1] * p.n[2]),
                                            d_sums);
  return 0;
}

int launch_init_eval(const InitArgs& A, const fvb_layout& L, const double* vecs, int ninst, double* out,
                     unsigned long long* bad, cudaStream_t st) {
  const int64_t n = A.n[0] * A.n[1] * A.n[2] * ninst;
  init_eval_kernel<<<grid_for(n), 256, 0, st>>>(A, L, vecs, ninst, out, bad);
  return 0;
}

}  // namespace fvb
