// knn_augmented row sampling for one tree level (skeleton.py:111-121).
//
// mark: every point's kNN list is OR-ed into its node's bitmap over [0, n),
// skipping neighbours inside the node -- np.unique of the union minus the
// node range, as a bitmap -- and the per-node counts go to the host, which
// makes the reference's RNG top-up draws (indices into
// rest = complement \ base, in ascending order).
// fill: the top-up ranks are mapped to points (r-th clear bit outside the
// node), set, and each node's set bits are compacted in ascending order.
#include <vector>

#include "hks_internal.h"

namespace hks {
namespace {

void level_ranges(int64_t n, int64_t level, std::vector<int64_t>& beg, std::vector<int64_t>& sz) {
  beg.assign(1, 0);
  sz.assign(1, n);
  for (int64_t l = 0; l < level; ++l) {
    std::vector<int64_t> nb, ns;
    for (size_t j = 0; j < beg.size(); ++j) {
      const int64_t half = (sz[j] + 1) / 2;  // tree.py:117
      nb.push_back(beg[j]);
      ns.push_back(half);
      nb.push_back(beg[j] + half);
      ns.push_back(sz[j] - half);
    }
    beg.swap(nb);
    sz.swap(ns);
  }
}

__device__ __forceinline__ int node_of(const int64_t* beg, int count, int64_t p) {
  int lo = 0, hi = count - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (beg[mid] <= p) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// knn holds the lists of the points [row0, row0 + nrows) (global indices);
// the bitmaps belong to `count` consecutive nodes of one level
__global__ void mark_kernel(const int64_t* __restrict__ knn, int64_t row0, int64_t nrows, int kappa,
                            const int64_t* __restrict__ beg, const int64_t* __restrict__ sz, int count, int64_t words,
                            unsigned* __restrict__ bm) {
  const int64_t lo = beg[0], hi = beg[count - 1] + sz[count - 1];
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nrows * kappa;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = row0 + e / kappa;
    if (p < lo || p >= hi) continue;
    const int j = node_of(beg, count, p);
    const int64_t q = knn[e];
    if (q >= beg[j] && q < beg[j] + sz[j]) continue;
    atomicOr(bm + (size_t)j * words + (q >> 5), 1u << (q & 31));
  }
}

__global__ void count_kernel(const unsigned* __restrict__ bm, int64_t words, int64_t* __restrict__ counts) {
  __shared__ double red[8];
  const unsigned* b = bm + (size_t)blockIdx.x * words;
  double c = 0.0;
  for (int64_t w = threadIdx.x; w < words; w += blockDim.x) c += __popc(b[w]);
  c = block_sum(c, red);
  if (threadIdx.x == 0) counts[blockIdx.x] = (int64_t)c;
}

// bits that are NOT available for the rest-set: node range, bits >= n
__device__ __forceinline__ unsigned blocked_bits(int64_t w, int64_t b, int64_t e, int64_t n) {
  unsigned m = 0;
  const int64_t lo = w * 32;
  for (int t = 0; t < 32; ++t) {
    const int64_t p = lo + t;
    if (p >= n || (p >= b && p < e)) m |= 1u << t;
  }
  return m;
}

// one CTA per node with top-up draws: prefix counts of free bits, then each
// draw r becomes the r-th free point (rest[r]) and is set in the bitmap
__global__ void topup_kernel(unsigned* __restrict__ bm, int64_t words, int64_t n, const int64_t* __restrict__ beg,
                             const int64_t* __restrict__ sz, const int* __restrict__ nodes,
                             const int64_t* __restrict__ extra, const int64_t* __restrict__ eoff,
                             int64_t* __restrict__ zpre_all, int64_t* __restrict__ posbuf) {
  const int j = nodes[blockIdx.x];
  unsigned* b = bm + (size_t)j * words;
  int64_t* zpre = zpre_all + (size_t)blockIdx.x * (words + 1);
  const int64_t nb = beg[j], ne = beg[j] + sz[j];
  if (threadIdx.x == 0) {  // sequential scan: only nodes short of samples get here
    int64_t acc = 0;
    for (int64_t w = 0; w < words; ++w) {
      zpre[w] = acc;
      acc += 32 - __popc(b[w] | blocked_bits(w, nb, ne, n));
    }
    zpre[words] = acc;
  }
  __syncthreads();
  // phase 1: map every draw against the ORIGINAL rest set (no bit is set
  // yet, so concurrent draws cannot shift each other's ranks)
  for (int64_t t = eoff[blockIdx.x] + threadIdx.x; t < eoff[blockIdx.x + 1]; t += blockDim.x) {
    const int64_t r = extra[t];
    int64_t lo = 0, hi = words - 1;  // last word with zpre <= r
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) >> 1;
      if (zpre[mid] <= r) lo = mid; else hi = mid - 1;
    }
    const unsigned freeb = ~(b[lo] | blocked_bits(lo, nb, ne, n));
    int64_t k = r - zpre[lo];
    int64_t pos = -1;
    for (int bit = 0; bit < 32; ++bit) {
      if (freeb & (1u << bit)) {
        if (k == 0) {
          pos = lo * 32 + bit;
          break;
        }
        --k;
      }
    }
    posbuf[t] = pos;
  }
  __syncthreads();
  // phase 2: add the drawn rows
  for (int64_t t = eoff[blockIdx.x] + threadIdx.x; t < eoff[blockIdx.x + 1]; t += blockDim.x) {
    const int64_t pos = posbuf[t];
    if (pos >= 0) atomicOr(b + (pos >> 5), 1u << (pos & 31));
  }
}

// one CTA per node: ascending compaction of the set bits
__global__ void compact_kernel(const unsigned* __restrict__ bm, int64_t words, const int64_t* __restrict__ roff,
                               int64_t* __restrict__ rows) {
  const unsigned* b = bm + (size_t)blockIdx.x * words;
  int64_t* out = rows + roff[blockIdx.x];
  __shared__ int64_t scan[1024];
  __shared__ int64_t base;
  if (threadIdx.x == 0) base = 0;
  __syncthreads();
  for (int64_t w0 = 0; w0 < words; w0 += blockDim.x) {
    const int64_t w = w0 + threadIdx.x;
    const unsigned bits = w < words ? b[w] : 0u;
    scan[threadIdx.x] = __popc(bits);
    __syncthreads();
    for (int o = 1; o < (int)blockDim.x; o <<= 1) {  // inclusive Hillis-Steele scan
      const int64_t v = threadIdx.x >= (unsigned)o ? scan[threadIdx.x - o] : 0;
      __syncthreads();
      scan[threadIdx.x] += v;
      __syncthreads();
    }
    int64_t pos = base + scan[threadIdx.x] - __popc(bits);
    for (int t = 0; t < 32; ++t)
      if (bits & (1u << t)) out[pos++] = w * 32 + t;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) base += scan[threadIdx.x];
    __syncthreads();
  }
}

}  // namespace
}  // namespace hks

using namespace hks;

namespace {
int subset_ranges(int64_t n, int64_t level, int64_t node0, int64_t count, std::vector<int64_t>& beg,
                  std::vector<int64_t>& sz) {
  if (level < 0 || level > 40 || node0 < 0 || count < 1 || node0 + count > ((int64_t)1 << level)) return -1;
  level_ranges(n, level, beg, sz);
  beg = std::vector<int64_t>(beg.begin() + node0, beg.begin() + node0 + count);
  sz = std::vector<int64_t>(sz.begin() + node0, sz.begin() + node0 + count);
  return 0;
}
}  // namespace

extern "C" int hks_knn_rows_mark_ex(const int64_t* knn, int64_t row0, int64_t nrows, int64_t n, int64_t kappa,
                                    int64_t level, int64_t node0, int64_t count_, int32_t* bitmap,
                                    int64_t* counts_host, void* stream) {
  std::vector<int64_t> beg, sz;
  if ((!knn && nrows > 0) || !bitmap || !counts_host || level < 1 || row0 < 0 || nrows < 0 || row0 + nrows > n ||
      subset_ranges(n, level, node0, count_, beg, sz))
    return set_error(HKS_ERR_INVALID, "hks_knn_rows_mark: bad arguments");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int count = (int)beg.size();
  const int64_t words = (n + 31) / 32;
  int64_t *dbeg = nullptr, *dsz = nullptr, *dcnt = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&dbeg), count * sizeof(int64_t), s);
  if (e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void**>(&dsz), count * sizeof(int64_t), s);
  if (e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void**>(&dcnt), count * sizeof(int64_t), s);
  if (e == cudaSuccess) {
    cudaMemcpyAsync(dbeg, beg.data(), count * sizeof(int64_t), cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(dsz, sz.data(), count * sizeof(int64_t), cudaMemcpyHostToDevice, s);
    cudaMemsetAsync(bitmap, 0, (size_t)count * words * sizeof(unsigned), s);
    if (nrows > 0)
      mark_kernel<<<1184, 256, 0, s>>>(knn, row0, nrows, (int)kappa, dbeg, dsz, count, words,
                                       reinterpret_cast<unsigned*>(bitmap));
    count_kernel<<<count, 256, 0, s>>>(reinterpret_cast<unsigned*>(bitmap), words, dcnt);
    e = cudaMemcpyAsync(counts_host, dcnt, count * sizeof(int64_t), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  }
  if (dbeg) cudaFreeAsync(dbeg, s);
  if (dsz) cudaFreeAsync(dsz, s);
  if (dcnt) cudaFreeAsync(dcnt, s);
  if (e != cudaSuccess) return set_error(HKS_ERR_CUDA, "hks_knn_rows_mark: %s", cudaGetErrorString(e));
  return HKS_OK;
}

extern "C" int hks_knn_rows_mark(const int64_t* knn, int64_t n, int64_t kappa, int64_t level, int64_t depth,
                                 int32_t* bitmap, int64_t* counts_host, void* stream) {
  if (level > depth) return set_error(HKS_ERR_INVALID, "hks_knn_rows_mark: bad arguments");
  return hks_knn_rows_mark_ex(knn, 0, n, n, kappa, level, 0, (int64_t)1 << level, bitmap, counts_host, stream);
}

extern "C" int hks_bitmap_count(const int32_t* bitmap, int64_t n, int64_t count, int64_t* counts_host, void* stream) {
  if (!bitmap || !counts_host || n < 1 || count < 1) return set_error(HKS_ERR_INVALID, "hks_bitmap_count: bad arguments");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t words = (n + 31) / 32;
  int64_t* dcnt = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&dcnt), count * sizeof(int64_t), s);
  if (e == cudaSuccess) {
    count_kernel<<<(unsigned)count, 256, 0, s>>>(reinterpret_cast<const unsigned*>(bitmap), words, dcnt);
    e = cudaMemcpyAsync(counts_host, dcnt, count * sizeof(int64_t), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    cudaFreeAsync(dcnt, s);
  }
  if (e != cudaSuccess) return set_error(HKS_ERR_CUDA, "hks_bitmap_count: %s", cudaGetErrorString(e));
  return HKS_OK;
}

extern "C" int hks_knn_rows_fill_ex(int64_t n, int64_t level, int64_t node0, int64_t count_, int32_t* bitmap,
                                    const int64_t* extra, const int64_t* extra_off_host, int64_t* rows,
                                    const int64_t* row_off_host, void* stream) {
  std::vector<int64_t> beg, sz;
  if (!bitmap || !rows || !extra_off_host || !row_off_host || level < 1 ||
      subset_ranges(n, level, node0, count_, beg, sz))
    return set_error(HKS_ERR_INVALID, "hks_knn_rows_fill: bad arguments");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int count = (int)beg.size();
  const int64_t words = (n + 31) / 32;
  std::vector<int> topup;
  std::vector<int64_t> eoff(1, 0);
  for (int j = 0; j < count; ++j) {
    const int64_t ne = extra_off_host[j + 1] - extra_off_host[j];
    if (ne > 0) {
      topup.push_back(j);
      eoff.push_back(eoff.back() + ne);
    }
  }
  cudaError_t e = cudaSuccess;
  int64_t *dbeg = nullptr, *dsz = nullptr, *deoff = nullptr, *dro = nullptr, *zpre = nullptr, *dextra = nullptr;
  int64_t* dpos = nullptr;
  int* dnodes = nullptr;
  e = cudaMallocAsync(reinterpret_cast<void**>(&dro), (count + 1) * sizeof(int64_t), s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dro, row_off_host, (count + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess && !topup.empty()) {
    const int nt = (int)topup.size();
    // the extra draws of the short nodes, contiguous in node order
    std::vector<int64_t> gather;
    e = cudaMallocAsync(reinterpret_cast<void**>(&dbeg), count * sizeof(int64_t), s);
    if (e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void**>(&dsz), count * sizeof(int64_t), s);
    if (e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void**>(&deoff), (nt + 1) * sizeof(int64_t), s);
    if (e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void**>(&dnodes), nt * sizeof(int), s);
    if (e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void**>(&zpre), (size_t)nt * (words + 1) * sizeof(int64_t), s);
    if (e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void**>(&dextra), eoff.back() * sizeof(int64_t), s);
    if (e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void**>(&dpos), eoff.back() * sizeof(int64_t), s);
    if (e == cudaSuccess) {
      cudaMemcpyAsync(dbeg, beg.data(), count * sizeof(int64_t), cudaMemcpyHostToDevice, s);
      cudaMemcpyAsync(dsz, sz.data(), count * sizeof(int64_t), cudaMemcpyHostToDevice, s);
      cudaMemcpyAsync(deoff, eoff.data(), (nt + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s);
      cudaMemcpyAsync(dnodes, topup.data(), nt * sizeof(int), cudaMemcpyHostToDevice, s);
      for (int t = 0; t < nt; ++t) {
        const int j = topup[t];
        cudaMemcpyAsync(dextra + eoff[t], extra + extra_off_host[j], (eoff[t + 1] - eoff[t]) * sizeof(int64_t),
                        cudaMemcpyDeviceToDevice, s);
      }
      topup_kernel<<<nt, 256, 0, s>>>(reinterpret_cast<unsigned*>(bitmap), words, n, dbeg, dsz, dnodes, dextra,
                                      deoff, zpre, dpos);
    }
  }
  if (e == cudaSuccess) {
    compact_kernel<<<count, 1024, 0, s>>>(reinterpret_cast<unsigned*>(bitmap), words, dro, rows);
    e = cudaGetLastError();
  }
  for (void* p : {(void*)dbeg, (void*)dsz, (void*)deoff, (void*)dro, (void*)zpre, (void*)dextra, (void*)dnodes,
                  (void*)dpos})
    if (p) cudaFreeAsync(p, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return set_error(HKS_ERR_CUDA, "hks_knn_rows_fill: %s", cudaGetErrorString(e));
  return HKS_OK;
}

extern "C" int hks_knn_rows_fill(int64_t n, int64_t level, int64_t depth, int32_t* bitmap, const int64_t* extra,
                                 const int64_t* extra_off_host, int64_t* rows, const int64_t* row_off_host,
                                 void* stream) {
  if (level > depth) return set_error(HKS_ERR_INVALID, "hks_knn_rows_fill: bad arguments");
  return hks_knn_rows_fill_ex(n, level, 0, (int64_t)1 << level, bitmap, extra, extra_off_host, rows, row_off_host,
                              stream);
}
