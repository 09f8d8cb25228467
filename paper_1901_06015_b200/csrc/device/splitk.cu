// Split-K for problems with too few CTA tiles to fill 148 SMs (small m x n):
// the fast kernels then give each tile's k-range to `splits` CTAs, which
// write their partial accumulator tiles to a workspace; this pass sums them
// in split order (deterministic, independent of scheduling) and runs the same
// fused typecast-accumulate epilogue as the single-pass kernels.
#include <cstdlib>

#include "common.cuh"

namespace mdg {
namespace {

constexpr int RED_THREADS = 256;

template <int CDT, typename AccT>
__global__ void __launch_bounds__(RED_THREADS)
    splitk_reduce_kernel(const __grid_constant__ GemmDesc d, int BM, int BN, uint32_t region) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* cbar = reinterpret_cast<uint64_t*>(smem + region);
  if (threadIdx.x == 0) {
    mbar_init(cbar, 1);
    mbar_fence_init();
  }
  __syncthreads();
  const int tiles_m = static_cast<int>((d.me + BM - 1) / BM);
  const int tiles_n = static_cast<int>((d.ne + BN - 1) / BN);
  const int64_t tiles = static_cast<int64_t>(tiles_m) * tiles_n;
  const int64_t tile_id = blockIdx.x;
  int tm, tn;
  tile_coords(tile_id, tiles_m, tiles_n, d.group_rows, tm, tn);
  const int elems = BM * BN;
  const AccT* base = static_cast<const AccT*>(d.partials) + tile_id * elems;
  const int64_t stride = tiles * elems;
  uint32_t cphase = 0;
  fast_epilogue<CDT>(smem, region, cbar, d.epi, static_cast<int64_t>(tm) * BM, static_cast<int64_t>(tn) * BN, BM, BN,
                     threadIdx.x, RED_THREADS, cphase, [&](auto&& put) {
                       for (int e = threadIdx.x; e < elems; e += RED_THREADS) {
                         AccT s = base[e];
                         for (int sp = 1; sp < d.splits; ++sp) s = s + base[sp * stride + e];
                         put(e % BM, e / BM, static_cast<double>(s));
                       }
                     });
}

}  // namespace

int choose_splits(int64_t tiles, int64_t nk, int slots) {
  if (const char* force = std::getenv("MDGEMM_SPLITK")) {  // tuning override: 0 = auto, n = force n
    const int f = std::atoi(force);
    if (f > 0) return static_cast<int>(std::min<int64_t>(f, nk));
  }
  // Measured on B200: 5-6x for small outputs with a long k (256x256x16384),
  // but a loss on small cubes (512^3, 1024^3) where the extra pass and the
  // partial traffic cost more than the idle SMs.  Split only when the grid is
  // at least 2x underfilled and every slice keeps >= 32 k-blocks (512 steps).
  if (tiles * 2 > slots || nk < 64) return 1;
  int64_t s = (slots + tiles - 1) / tiles;  // enough CTAs for one full wave
  s = std::min<int64_t>(s, nk / 32);
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(s, 16)));
}

cudaError_t launch_splitk_reduce(const GemmDesc& d, const FastTile& t, bool single, cudaStream_t s) {
  const int64_t tiles = ((d.me + t.bm - 1) / t.bm) * ((d.ne + t.bn - 1) / t.bn);
  if (tiles == 0 || d.splits <= 1) return cudaSuccess;
  const uint32_t region = static_cast<uint32_t>(t.bm) * t.bn * 8 * 3 / 2;
  const size_t smem = region + sizeof(uint64_t);
  cudaError_t e = cudaSuccess;
  MDG_DISPATCH_CDT(d.epi.out.dtype, CDT, {
    if (single) {
      e = cudaFuncSetAttribute(splitk_reduce_kernel<CDT, float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(smem));
      if (e != cudaSuccess) return e;
      splitk_reduce_kernel<CDT, float><<<static_cast<unsigned>(tiles), RED_THREADS, smem, s>>>(d, t.bm, t.bn, region);
    } else {
      e = cudaFuncSetAttribute(splitk_reduce_kernel<CDT, double>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(smem));
      if (e != cudaSuccess) return e;
      splitk_reduce_kernel<CDT, double><<<static_cast<unsigned>(tiles), RED_THREADS, smem, s>>>(d, t.bm, t.bn, region);
    }
  });
  return cudaGetLastError();
}

}  // namespace mdg
