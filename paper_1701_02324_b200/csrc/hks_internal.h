// Internal (C++) interface between the kernel translation units and the C-ABI.
#pragma once

#include <cstdarg>
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/hks.h"
#include "common.cuh"

namespace hks {

// Device copy of a base table for one-off launches (stream-ordered upload
// from host memory; free with cudaFreeAsync).
cudaError_t upload_bases(const Bases& b, Bases** dev, cudaStream_t s);

// Raise (never lower) a kernel's dynamic shared-memory limit.  Launches
// with different smem sizes share one function attribute; lowering it after
// a larger launch was captured into a CUDA graph makes that node invalid.
cudaError_t raise_smem_limit(const void* func, size_t bytes);
template <class F>
inline cudaError_t raise_smem_limit(F* func, size_t bytes) {
  return raise_smem_limit(reinterpret_cast<const void*>(func), bytes);
}

// Records a thread-local error message (read back through hks_last_error)
// and returns `code` so call sites can `return set_error(...)`.
int set_error(int code, const char* fmt, ...);

cudaError_t launch_gemm_batched(const Bases* bases, const GemmDesc* d_descs, int count, int max_m,
                                int max_n, cudaStream_t stream);
cudaError_t launch_copy_batched(const Bases* bases, const CopyDesc* d_descs, int count, int max_elems,
                                cudaStream_t stream);
cudaError_t launch_getrf_batched(const Bases* bases, const LuDesc* d_descs, int count, int max_n,
                                 cudaStream_t stream);
cudaError_t launch_getrs_batched(const Bases* bases, const LuSolveDesc* d_descs, int count, int max_n,
                                 int max_nrhs, cudaStream_t stream);
cudaError_t launch_panel_batched(const Bases* b, const PanelDesc* d, int count, int max_rows, int pb,
                                 cudaStream_t s);
cudaError_t launch_swap_batched(const Bases* b, const SwapDesc* d, int count, int max_cols, cudaStream_t s);
cudaError_t launch_getrs_fused(const Bases* b, const GetrsDesc* d, int count, int max_n, int max_cols,
                               cudaStream_t s);
cudaError_t launch_gather_batched(const Bases* b, const GatherDesc* d, int count, int max_rows, int max_cols,
                                  cudaStream_t s);
cudaError_t launch_trsm_batched(const Bases* b, const TrsmDesc* d, int count, int max_cols, int max_k, bool upper,
                                cudaStream_t s);
cudaError_t launch_lu_fused(const Bases* b, const LuFusedDesc* d, int count, int max_n, int max_r,
                            cudaStream_t s);
cudaError_t launch_norm1_batched(const Bases* b, const LuDesc* d, int count, cudaStream_t s);

// Tall-skinny QR pre-reduction (tsqr.cu): R (c x c, row-major, upper
// triangular, initially zero or a previous result) absorbs the nrows rows of
// S (row-major, ld lds; destroyed).  tri != 0: S is itself upper triangular.
struct TsqrJob {
  double* R;
  double* S;
  int c, lds, nrows, tri;
};
int tsqr_slab_rows();
cudaError_t launch_tsqr_absorb(const TsqrJob* d_jobs, int count, cudaStream_t s);
// dgecon estimates; phase -1: one monolithic launch; phase 0..kGeconSteps:
// the split estimate (init, then one LU application + dlacn2 step per
// launch) with per-matrix state in base kGeconScratchBase.
constexpr int kGeconSteps = 11;      // dlacn2 applies A, B, 4 x (C, D), E
constexpr int kGeconScratchBase = 14;  // == B_VWS (plan.h)
inline int gecon_stride(int max_n) { return 2 * (max_n > 0 ? max_n : 1) + 8; }
cudaError_t launch_gecon_batched(const Bases* bases, const LuDesc* d_descs, int count, int max_n,
                                 cudaStream_t stream, int phase = -1);

// Kernel-block evaluation (K1/K2/K3).  Rows/cols are either explicit global
// (tree-order) index lists or contiguous ranges starting at row0/col0.
struct EvalDesc {
  Ref rows;  // int64 index list, or kNull for the range row0 + [0, m)
  Ref cols;
  int64_t row0, col0;
  int m, n;
  Ref out;
  int ldo;
  int diag;  // add Bases::lam where the local row index equals the local column index
};

struct KernelParams {
  int family;     // HKS_GAUSSIAN / HKS_LAPLACE3D / HKS_POLYNOMIAL
  double h;       // gaussian bandwidth
  double neg2h2;  // -2 h^2, formed as in kernels.py:95
  int degree;
  double shift;
};

KernelParams make_kernel_params(const hks_kernel* k);

cudaError_t launch_eval_batched(const double* X, int d, KernelParams kp, const Bases* bases,
                                const EvalDesc* d_descs, int count, int max_m, int max_n, bool row_major,
                                cudaStream_t stream);

// U[i,:] = beta*U[i,:] + sum_j K(x_rows[i], x_cols[j]) W[j,:] + diag * W[i,:]
// (the diag term only when rows and cols are the same range), never
// materialising K: the fused kernel-summation used by hmatvec's leaf level
// and by the sampled accuracy checks.
struct SumDesc {
  Ref rows;
  Ref cols;
  int64_t row0, col0;
  int m, n, k;
  Ref W;
  int ldw;
  Ref U;
  int ldu;
  double beta;
  int diag;  // add Bases::lam * W (rows == cols ranges only)
};

cudaError_t launch_ksum_batched(const double* X, int d, KernelParams kp, const Bases* bases,
                                const SumDesc* d_descs, int count, int max_m, cudaStream_t stream,
                                const double* XC = nullptr);

}  // namespace hks
