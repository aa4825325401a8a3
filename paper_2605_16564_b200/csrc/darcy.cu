// darcy.cu — the P1 pressure solve that consumes a surrogate (SURVEY §8f row 2,
// reference darcy.py:238-375): deterministic stiffness assembly and a
// Jacobi-preconditioned conjugate-gradient solve on the device.
//
// Assembly: the host builds the CSR pattern of A and, per nonzero, the list
// of element contributions in the reference's COO order (rows = repeat(tris),
// cols = tile(tris), darcy.py:330-332); the kernel sums them in that order
// with round-to-nearest arithmetic, so every entry is bit-identical to the
// reference's COO -> CSR duplicate sum.  2D local matrix (darcy.py:322-328):
// (b_i b_j + c_i c_j) * (k / (4 A)); 1D (darcy.py:359-363): +-k/h.
//
// PCG: the loop of scipy.sparse.linalg.cg (M = diag(1/a_ii), x0 = 0, stop when
// ||r|| < rtol ||b|| checked before each iteration) with every vector in HBM
// and every scalar in device memory; dot products are fixed-order two-stage
// reductions (run-to-run deterministic).  A device flag stops the iteration
// so the host only polls it every PCG_POLL iterations.
#include "pam_common.cuh"

#include <algorithm>
#include <vector>

namespace pam {

__global__ void p1_values_kernel(int dim, int64_t nnz, const int64_t* __restrict__ slot_ptr,
                                 const int64_t* __restrict__ contrib,
                                 const int64_t* __restrict__ elem_nodes, const double* __restrict__ nodes,
                                 const double* __restrict__ coef, double* __restrict__ values) {
  const int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= nnz) return;
  double acc = 0.0;
  bool first = true;
  for (int64_t q = slot_ptr[s]; q < slot_ptr[s + 1]; ++q) {
    const int64_t c = contrib[q];
    double v;
    if (dim == 2) {
      const int64_t e = c / 9;
      const int i = static_cast<int>((c % 9) / 3), j = static_cast<int>(c % 3);
      const int64_t* t = elem_nodes + 3 * e;
      const double x0 = nodes[2 * t[0]], y0 = nodes[2 * t[0] + 1];
      const double x1 = nodes[2 * t[1]], y1 = nodes[2 * t[1] + 1];
      const double x2 = nodes[2 * t[2]], y2 = nodes[2 * t[2] + 1];
      const double bv[3] = {__dsub_rn(y1, y2), __dsub_rn(y2, y0), __dsub_rn(y0, y1)};
      const double cv[3] = {__dsub_rn(x2, x1), __dsub_rn(x0, x2), __dsub_rn(x1, x0)};
      // area: 0.5 * (d1x * d2y - d1y * d2x) with d1 = p1 - p0, d2 = p2 - p0 (darcy.py:52-56)
      const double area = __dmul_rn(0.5, __dsub_rn(__dmul_rn(__dsub_rn(x1, x0), __dsub_rn(y2, y0)),
                                                   __dmul_rn(__dsub_rn(y1, y0), __dsub_rn(x2, x0))));
      const double scale = __ddiv_rn(coef[e], __dmul_rn(4.0, area));
      v = __dmul_rn(__dadd_rn(__dmul_rn(bv[i], bv[j]), __dmul_rn(cv[i], cv[j])), scale);
    } else {
      const int64_t e = c / 4;
      const int i = static_cast<int>((c % 4) / 2), j = static_cast<int>(c % 2);
      const double h = __dsub_rn(nodes[e + 1], nodes[e]);
      const double w = __ddiv_rn(coef[e], h);
      v = (i == j) ? w : -w;
    }
    acc = first ? v : __dadd_rn(acc, v);
    first = false;
  }
  values[s] = acc;
}

__global__ void spmv_kernel(int64_t n, const int64_t* __restrict__ row_ptr, const int64_t* __restrict__ col,
                            const double* __restrict__ val, const double* __restrict__ x,
                            double* __restrict__ y) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double acc = 0.0;
  for (int64_t q = row_ptr[i]; q < row_ptr[i + 1]; ++q) acc = fma(val[q], x[col[q]], acc);
  y[i] = acc;
}

// ---- PCG -----------------------------------------------------------------
constexpr int CG_THREADS = 256;
constexpr int PCG_POLL = 16;

struct CgState {      // device scalars
  double atol;        // rtol * ||b||
  double rho_prev;
  double beta;
  double alpha;
  double rr;          // ||r||^2 of the last check
  int64_t it;         // completed iterations
  int64_t done;       // 1 = converged, 2 = maxiter
};

// fixed-order block reduction of up to 2 values; one partial pair per block
__device__ __forceinline__ void block_sum2(double a, double b, double* part) {
  __shared__ double sa[CG_THREADS], sb[CG_THREADS];
  sa[threadIdx.x] = a;
  sb[threadIdx.x] = b;
  __syncthreads();
  for (int o = CG_THREADS / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      sa[threadIdx.x] += sa[threadIdx.x + o];
      sb[threadIdx.x] += sb[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = sa[0];
    part[2 * blockIdx.x + 1] = sb[0];
  }
}

__global__ void cg_diag_kernel(int64_t n, const int64_t* __restrict__ row_ptr, const int64_t* __restrict__ col,
                               const double* __restrict__ val, double* __restrict__ dinv) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double d = 0.0;
  for (int64_t q = row_ptr[i]; q < row_ptr[i + 1]; ++q)
    if (col[q] == i) d += val[q];
  dinv[i] = d > 0.0 ? 1.0 / d : 1.0;  // np.where(diag > 0, 1/diag, 1) (darcy.py:277)
}

// (first call) or: x += alpha p; r -= alpha q; then z = M r, partials (r.r, r.z)
__global__ void cg_update_kernel(int64_t n, int first, const CgState* st, double* __restrict__ x,
                                 double* __restrict__ r, const double* __restrict__ p,
                                 const double* __restrict__ q, const double* __restrict__ dinv,
                                 double* __restrict__ z, double* part) {
  if (st->done) return;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  double rr = 0.0, rz = 0.0;
  if (i < n) {
    double ri = r[i];
    if (!first) {
      const double al = st->alpha;
      x[i] = __dadd_rn(x[i], __dmul_rn(al, p[i]));
      ri = __dsub_rn(ri, __dmul_rn(al, q[i]));
      r[i] = ri;
    }
    const double zi = __dmul_rn(dinv[i], ri);
    z[i] = zi;
    rr = ri * ri;
    rz = ri * zi;
  }
  block_sum2(rr, rz, part);
}

// convergence check (before the iteration, as scipy) and beta
__global__ void cg_check_kernel(int nblk, int64_t max_iter, CgState* st, const double* part) {
  if (st->done || threadIdx.x != 0) return;
  double rr = 0.0, rz = 0.0;
  for (int b = 0; b < nblk; ++b) {
    rr += part[2 * b];
    rz += part[2 * b + 1];
  }
  st->rr = rr;
  if (st->it >= max_iter) {  // scipy returns info = maxiter without a final check
    st->done = 2;
    return;
  }
  if (sqrt(rr) < st->atol) {
    st->done = 1;
    return;
  }
  st->beta = (st->it > 0) ? rz / st->rho_prev : 0.0;
  st->rho_prev = rz;
}

// p = z (first) or p = beta p + z (p *= beta; p += z)
__global__ void cg_dir_kernel(int64_t n, const CgState* st, double* __restrict__ p, const double* __restrict__ z) {
  if (st->done) return;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  p[i] = (st->it > 0) ? __dadd_rn(__dmul_rn(st->beta, p[i]), z[i]) : z[i];
}

// q = A p and partial p.q
__global__ void cg_spmv_kernel(int64_t n, const CgState* st, const int64_t* __restrict__ row_ptr,
                               const int64_t* __restrict__ col, const double* __restrict__ val,
                               const double* __restrict__ p, double* __restrict__ q, double* part) {
  if (st->done) return;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  double pq = 0.0;
  if (i < n) {
    double acc = 0.0;
    for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) acc = fma(val[k], p[col[k]], acc);
    q[i] = acc;
    pq = p[i] * acc;
  }
  block_sum2(pq, 0.0, part);
}

__global__ void cg_alpha_kernel(int nblk, CgState* st, const double* part) {
  if (st->done || threadIdx.x != 0) return;
  double pq = 0.0;
  for (int b = 0; b < nblk; ++b) pq += part[2 * b];
  st->alpha = st->rho_prev / pq;
  st->it += 1;
}

__global__ void cg_init_kernel(int nblk, double rtol, CgState* st, const double* part) {
  if (threadIdx.x != 0) return;
  double bb = 0.0;
  for (int b = 0; b < nblk; ++b) bb += part[2 * b];
  st->atol = rtol * sqrt(bb);
  st->rho_prev = 0.0;
  st->beta = 0.0;
  st->alpha = 0.0;
  st->rr = bb;
  st->it = 0;
  st->done = (bb == 0.0) ? 1 : 0;
}

__global__ void sumsq_kernel(int64_t n, const double* __restrict__ v, double* part) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const double a = (i < n) ? v[i] : 0.0;
  block_sum2(a * a, 0.0, part);
}

}  // namespace pam

using namespace pam;

extern "C" int pam_p1_values_f64(int dim, int64_t nnz, const int64_t* slot_ptr, const int64_t* contrib,
                                 const int64_t* elem_nodes, const double* nodes, const double* coef,
                                 double* values, void* stream) {
  if ((dim != 1 && dim != 2) || nnz < 0) return PAM_ERR_ARG;
  if (nnz == 0) return PAM_OK;
  p1_values_kernel<<<(unsigned)ceil_div(nnz, 256), 256, 0, as_stream(stream)>>>(
      dim, nnz, slot_ptr, contrib, elem_nodes, nodes, coef, values);
  PAM_LAUNCH_CHECK("p1_values_kernel");
  return PAM_OK;
}

extern "C" int pam_csr_spmv_f64(int64_t n, const int64_t* row_ptr, const int64_t* col, const double* val,
                                const double* x, double* y, void* stream) {
  if (n < 0) return PAM_ERR_ARG;
  if (n == 0) return PAM_OK;
  spmv_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, as_stream(stream)>>>(n, row_ptr, col, val, x, y);
  PAM_LAUNCH_CHECK("spmv_kernel");
  return PAM_OK;
}

extern "C" int64_t pam_pcg_workspace_bytes(int64_t n) {
  const int64_t nblk = ceil_div(std::max<int64_t>(n, 1), CG_THREADS);
  return (5 * n + 2 * nblk) * 8 + 256;
}

extern "C" int pam_pcg_f64(int64_t n, const int64_t* row_ptr, const int64_t* col, const double* val,
                           const double* b, double* x, double rtol, int64_t max_iter, void* work,
                           int64_t* iterations, int32_t* converged, double* rel_residual, void* stream) {
  if (n < 0 || rtol < 0.0 || max_iter < 0 || !work) return PAM_ERR_ARG;
  if (n == 0) {
    *iterations = 0;
    *converged = 1;
    *rel_residual = 0.0;
    return PAM_OK;
  }
  cudaStream_t s = as_stream(stream);
  const int64_t nblk64 = ceil_div(n, CG_THREADS);
  if (nblk64 > (1 << 30)) return PAM_ERR_UNSUPPORTED;
  const int nblk = static_cast<int>(nblk64);
  char* w = static_cast<char*>(work);
  CgState* st = reinterpret_cast<CgState*>(w);
  double* r = reinterpret_cast<double*>(w + 256);
  double* p = r + n;
  double* q = p + n;
  double* z = q + n;
  double* dinv = z + n;
  double* part = dinv + n;
  const unsigned g = static_cast<unsigned>(nblk);
  // x0 = 0, r = b (scipy: r = b.copy() when x0 is all zero)
  PAM_CUDA_CHECK(cudaMemsetAsync(x, 0, n * sizeof(double), s));
  PAM_CUDA_CHECK(cudaMemcpyAsync(r, b, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
  cg_diag_kernel<<<g, CG_THREADS, 0, s>>>(n, row_ptr, col, val, dinv);
  sumsq_kernel<<<g, CG_THREADS, 0, s>>>(n, b, part);
  cg_init_kernel<<<1, 32, 0, s>>>(nblk, rtol, st, part);
  PAM_LAUNCH_CHECK("pcg init");
  CgState h{};
  int64_t launched = 0;
  for (;;) {
    for (int k = 0; k < PCG_POLL; ++k, ++launched) {
      cg_update_kernel<<<g, CG_THREADS, 0, s>>>(n, launched == 0, st, x, r, p, q, dinv, z, part);
      cg_check_kernel<<<1, 32, 0, s>>>(nblk, max_iter, st, part);
      cg_dir_kernel<<<g, CG_THREADS, 0, s>>>(n, st, p, z);
      cg_spmv_kernel<<<g, CG_THREADS, 0, s>>>(n, st, row_ptr, col, val, p, q, part);
      cg_alpha_kernel<<<1, 32, 0, s>>>(nblk, st, part);
    }
    PAM_LAUNCH_CHECK("pcg iteration");
    PAM_CUDA_CHECK(cudaMemcpyAsync(&h, st, sizeof(CgState), cudaMemcpyDeviceToHost, s));
    PAM_CUDA_CHECK(cudaStreamSynchronize(s));
    if (h.done) break;
  }
  *iterations = h.it;
  *converged = (h.done == 1) ? 1 : 0;
  *rel_residual = (h.atol > 0.0 && rtol > 0.0) ? sqrt(h.rr) / (h.atol / rtol) : sqrt(h.rr);
  return PAM_OK;
}
