// Level-synchronous partition-tree build on the GPU (tree.py:70-144).
//
// For every level all nodes are processed together: per-node mean,
// `steps` normalised power iterations of the centred second moment from the
// caller's start vectors (the reference's default_rng([seed, level, begin])
// draws, made on the host), projection of the *uncentred* points on the
// direction, a stable per-node argsort (two stable LSD radix passes: key,
// then node id -- np.argsort(kind="stable") semantics, -0.0 == +0.0), the
// physical permutation of points and `perm`, and split_value =
// proj[local[half - 1]].  Reductions use fixed chunking, so the build is
// deterministic run to run.
#include <cub/device/device_radix_sort.cuh>
#include <algorithm>
#include <vector>

#include "hks_internal.h"

namespace hks {
namespace {

constexpr int CH = 2048;  // points per chunk (chunks never straddle nodes)
constexpr int TB = 256;

struct Chunk {
  int64_t begin, end;
  int node;  // local index within the level
  int pad;
};

// partial[c][k]: MEAN -> sum_p x_pk ; POWER -> sum_p u_p (x_pk - mu_k),
// u_p = (x_p - mu) . v
__global__ void __launch_bounds__(TB) accum_kernel(const double* __restrict__ X, int d,
                                                   const Chunk* __restrict__ chunks, int power,
                                                   const double* __restrict__ mean,
                                                   const double* __restrict__ v,
                                                   double* __restrict__ partial) {
  const Chunk c = chunks[blockIdx.x];
  __shared__ double u[CH];
  __shared__ double red[TB];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const double* mu = mean ? mean + (size_t)c.node * d : nullptr;
  const double* vv = v ? v + (size_t)c.node * d : nullptr;
  const int np = (int)(c.end - c.begin);
  if (power) {
    for (int p = wid; p < np; p += TB / 32) {
      const double* xp = X + (size_t)(c.begin + p) * d;
      double s = 0.0;
      for (int k = lane; k < d; k += 32) s = fma(xp[k] - mu[k], vv[k], s);
      s = warp_sum(s);
      if (lane == 0) u[p] = s;
    }
    __syncthreads();
  }
  // dims across td lanes, point groups across the rest
  const int td = d <= 32 ? 32 : TB, groups = TB / td;
  const int tk = threadIdx.x % td, tg = threadIdx.x / td;
  for (int k0 = 0; k0 < d; k0 += td) {
    const int k = k0 + tk;
    double acc = 0.0;
    if (k < d) {
      for (int p = tg; p < np; p += groups) {
        const double x = X[(size_t)(c.begin + p) * d + k];
        acc += power ? u[p] * (x - mu[k]) : x;
      }
    }
    red[threadIdx.x] = acc;
    __syncthreads();
    if (tg == 0 && k < d) {
      double s = 0.0;
      for (int g = 0; g < groups; ++g) s += red[g * td + tk];
      partial[(size_t)blockIdx.x * d + k] = s;
    }
    __syncthreads();
  }
}

// one CTA per node: MEAN -> mean = sum / size ; POWER -> v = w / ||w||
__global__ void __launch_bounds__(TB) node_reduce_kernel(const double* __restrict__ partial, int d,
                                                         const int* __restrict__ cfirst,
                                                         const int* __restrict__ ccount,
                                                         const int64_t* __restrict__ size, int power,
                                                         double* __restrict__ out, int* __restrict__ stopped,
                                                         double* __restrict__ wtmp) {
  const int j = blockIdx.x;
  __shared__ double red[TB / 32];
  if (power && stopped[j]) return;
  double* w = wtmp + (size_t)j * d;
  double ss = 0.0;
  for (int k = threadIdx.x; k < d; k += blockDim.x) {
    double s = 0.0;
    for (int c = 0; c < ccount[j]; ++c) s += partial[(size_t)(cfirst[j] + c) * d + k];
    if (power) {
      w[k] = s;
      ss = fma(s, s, ss);
    } else {
      out[(size_t)j * d + k] = s / (double)size[j];
    }
  }
  if (!power) return;
  const double nrm = sqrt(block_sum(ss, red));
  if (nrm == 0.0) {  // all points coincide: keep the direction (tree.py:81-82)
    if (threadIdx.x == 0) stopped[j] = 1;
    return;
  }
  for (int k = threadIdx.x; k < d; k += blockDim.x) out[(size_t)j * d + k] = w[k] / nrm;
}

__device__ __forceinline__ uint64_t order_key(double v) {
  if (v == 0.0) v = 0.0;  // -0.0 sorts equal to +0.0, like numpy's comparison sort
  const uint64_t b = __double_as_longlong(v);
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}

__global__ void project_kernel(const double* __restrict__ X, int d, const Chunk* __restrict__ chunks,
                               const double* __restrict__ v, double* __restrict__ proj,
                               uint64_t* __restrict__ keys, int* __restrict__ seg, int64_t* __restrict__ idx) {
  const Chunk c = chunks[blockIdx.x];
  const double* vv = v + (size_t)c.node * d;
  for (int64_t p = c.begin + threadIdx.x; p < c.end; p += blockDim.x) {
    const double* xp = X + (size_t)p * d;
    double s = 0.0;
    for (int k = 0; k < d; ++k) s = fma(xp[k], vv[k], s);
    proj[p] = s;
    keys[p] = order_key(s);
    seg[p] = c.node;
    idx[p] = p;
  }
}

__global__ void gather_seg(const int* __restrict__ seg, const int64_t* __restrict__ idx, int* __restrict__ out,
                           int64_t n) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x)
    out[p] = seg[idx[p]];
}

__global__ void permute_kernel(const double* __restrict__ Xo, const int64_t* __restrict__ po,
                               const double* __restrict__ proj, const int64_t* __restrict__ idx, int d, int64_t n,
                               double* __restrict__ Xn, int64_t* __restrict__ pn, double* __restrict__ projs) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = idx[p];
    pn[p] = po[s];
    projs[p] = proj[s];
    for (int k = 0; k < d; ++k) Xn[(size_t)p * d + k] = Xo[(size_t)s * d + k];
  }
}

__global__ void split_kernel(const double* __restrict__ projs, const int64_t* __restrict__ begin,
                             const int64_t* __restrict__ size, int count, const double* __restrict__ v, int d,
                             double* __restrict__ dirs_out, double* __restrict__ vals_out) {
  const int j = blockIdx.x;
  if (j >= count) return;
  for (int k = threadIdx.x; k < d; k += blockDim.x) dirs_out[(size_t)j * d + k] = v[(size_t)j * d + k];
  if (threadIdx.x == 0) {
    const int64_t half = (size[j] + 1) / 2;
    vals_out[j] = projs[begin[j] + half - 1];
  }
}

__global__ void iota64(int64_t* p, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = i;
}

template <class T>
struct Scratch {
  T* p = nullptr;
  cudaStream_t s;
  explicit Scratch(size_t n, cudaStream_t st, cudaError_t* e) : s(st) {
    cudaError_t r = cudaMallocAsync(reinterpret_cast<void**>(&p), (n ? n : 1) * sizeof(T), st);
    if (r != cudaSuccess && *e == cudaSuccess) *e = r;
  }
  ~Scratch() {
    if (p) cudaFreeAsync(p, s);
  }
};

}  // namespace
}  // namespace hks

using namespace hks;

// build_tree (tree.py:87-144).  X_in: n x d input-order points; starts:
// (2^depth - 1) x d normalised start vectors (heap order); outputs: X_out
// (tree order), perm_out, split_dirs ((2^depth - 1) x d), split_vals.
extern "C" int hks_build_tree(const double* X_in, int64_t n, int64_t d, int64_t depth, int64_t steps,
                              const double* starts, double* X_out, int64_t* perm_out, double* split_dirs,
                              double* split_vals, void* stream) {
  if (!X_in || !X_out || !perm_out || n < 1 || d < 1 || depth < 0)
    return set_error(HKS_ERR_INVALID, "hks_build_tree: bad arguments");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaSuccess;
  const int dd = (int)d;
  Scratch<double> Xa(n * d, s, &e), proj(n, s, &e), projs(n, s, &e);
  Scratch<int64_t> pa(n, s, &e), idx(n, s, &e), idx2(n, s, &e), idx3(n, s, &e);
  Scratch<uint64_t> keys(n, s, &e), keys2(n, s, &e);
  Scratch<int> seg(n, s, &e), seg2(n, s, &e), seg3(n, s, &e);
  if (e != cudaSuccess) return set_error(HKS_ERR_CUDA, "hks_build_tree: %s", cudaGetErrorString(e));
  // current arrays live in X_out / perm_out; Xa / pa are the other buffer
  double* Xc = X_out;
  double* Xn = Xa.p;
  int64_t* pc = perm_out;
  int64_t* pn = pa.p;
  e = cudaMemcpyAsync(Xc, X_in, n * d * sizeof(double), cudaMemcpyDeviceToDevice, s);
  iota64<<<256, 256, 0, s>>>(pc, n);
  size_t temp_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, temp_bytes, keys.p, keys2.p, idx.p, idx2.p, (int)n, 0, 64, s);
  size_t tb2 = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb2, seg2.p, seg3.p, idx2.p, idx3.p, (int)n, 0, 32, s);
  temp_bytes = std::max(temp_bytes, tb2);
  Scratch<char> temp(temp_bytes, s, &e);

  for (int64_t lev = 0; lev < depth && e == cudaSuccess; ++lev) {
    const int count = 1 << lev;
    // node ranges of this level (tree.py:117: left child takes ceil(size/2))
    std::vector<int64_t> beg(1, 0), sz(1, n);
    for (int64_t l = 0; l < lev; ++l) {
      std::vector<int64_t> nb, ns;
      for (size_t j = 0; j < beg.size(); ++j) {
        const int64_t half = (sz[j] + 1) / 2;
        nb.push_back(beg[j]);
        ns.push_back(half);
        nb.push_back(beg[j] + half);
        ns.push_back(sz[j] - half);
      }
      beg.swap(nb);
      sz.swap(ns);
    }
    std::vector<Chunk> ch;
    std::vector<int> cfirst(count), ccount(count);
    for (int j = 0; j < count; ++j) {
      cfirst[j] = (int)ch.size();
      for (int64_t b = beg[j]; b < beg[j] + sz[j]; b += CH)
        ch.push_back(Chunk{b, std::min(b + CH, beg[j] + sz[j]), j, 0});
      ccount[j] = (int)ch.size() - cfirst[j];
    }
    const int nch = (int)ch.size();
    Scratch<Chunk> dch(nch, s, &e);
    Scratch<int> dcf(count, s, &e), dcc(count, s, &e), stopped(count, s, &e);
    Scratch<int64_t> dbeg(count, s, &e), dsz(count, s, &e);
    Scratch<double> part((size_t)nch * d, s, &e), mean((size_t)count * d, s, &e), v((size_t)count * d, s, &e),
        wtmp((size_t)count * d, s, &e);
    if (e != cudaSuccess) break;
    cudaMemcpyAsync(dch.p, ch.data(), nch * sizeof(Chunk), cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(dcf.p, cfirst.data(), count * sizeof(int), cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(dcc.p, ccount.data(), count * sizeof(int), cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(dbeg.p, beg.data(), count * sizeof(int64_t), cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(dsz.p, sz.data(), count * sizeof(int64_t), cudaMemcpyHostToDevice, s);
    cudaMemsetAsync(stopped.p, 0, count * sizeof(int), s);
    const int64_t first = ((int64_t)1 << lev) - 1;
    if (d == 1) {  // tree.py:73-74: the direction is +1, no power steps
      std::vector<double> ones(count, 1.0);
      cudaMemcpyAsync(v.p, ones.data(), count * sizeof(double), cudaMemcpyHostToDevice, s);
    } else {
      cudaMemcpyAsync(v.p, starts + first * d, (size_t)count * d * sizeof(double), cudaMemcpyDeviceToDevice, s);
      accum_kernel<<<nch, TB, 0, s>>>(Xc, dd, dch.p, 0, nullptr, nullptr, part.p);
      node_reduce_kernel<<<count, TB, 0, s>>>(part.p, dd, dcf.p, dcc.p, dsz.p, 0, mean.p, stopped.p, wtmp.p);
      for (int64_t it = 0; it < steps; ++it) {  // tree.py:78-83
        accum_kernel<<<nch, TB, 0, s>>>(Xc, dd, dch.p, 1, mean.p, v.p, part.p);
        node_reduce_kernel<<<count, TB, 0, s>>>(part.p, dd, dcf.p, dcc.p, dsz.p, 1, v.p, stopped.p, wtmp.p);
      }
    }
    project_kernel<<<nch, TB, 0, s>>>(Xc, dd, dch.p, v.p, proj.p, keys.p, seg.p, idx.p);
    size_t tb = temp_bytes;
    cub::DeviceRadixSort::SortPairs(temp.p, tb, keys.p, keys2.p, idx.p, idx2.p, (int)n, 0, 64, s);
    gather_seg<<<592, 256, 0, s>>>(seg.p, idx2.p, seg2.p, n);
    int bits = 1;
    while ((1 << bits) < count) ++bits;
    tb = temp_bytes;
    cub::DeviceRadixSort::SortPairs(temp.p, tb, seg2.p, seg3.p, idx2.p, idx3.p, (int)n, 0, bits, s);
    permute_kernel<<<592, 256, 0, s>>>(Xc, pc, proj.p, idx3.p, dd, n, Xn, pn, projs.p);
    split_kernel<<<count, 64, 0, s>>>(projs.p, dbeg.p, dsz.p, count, v.p, dd, split_dirs + first * d,
                                      split_vals + first);
    std::swap(Xc, Xn);
    std::swap(pc, pn);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess && Xc != X_out) {
    e = cudaMemcpyAsync(X_out, Xc, n * d * sizeof(double), cudaMemcpyDeviceToDevice, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(perm_out, pc, n * sizeof(int64_t), cudaMemcpyDeviceToDevice, s);
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return set_error(HKS_ERR_CUDA, "hks_build_tree: %s", cudaGetErrorString(e));
  return HKS_OK;
}
