// Issue-rate microbenchmarks: the roofline denominators for the CUDA-core
// kernels (MEASURED_PEAKS.json only holds HBM and tensor-core peaks).
//
// k_peak_fsetp: 8 independent predicate chains of `setp.{lt,gt}.or.f32` --
//   the dom_tile inner loop without its loads/ballots -- 64 compares per
//   iteration per thread (+ 8 selp to keep the chains live).
// k_peak_fp32:  8 independent chains of mul.rn + add.rn (no FMA, like the
//   canonical association dot product): 16 flops per chain-step.
// k_peak_smem:  conflict-free ld.shared.v4 (each warp reads 512 contiguous
//   bytes per instruction) from a 32 KB array: shared-memory load bandwidth,
//   the bound of the rank-mask dominance sweep (k_dom_rank.cu).
#include "mo_common.cuh"

namespace mo {

__global__ void __launch_bounds__(256) k_peak_fsetp(const float* __restrict__ in, int iters, unsigned* out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  float a0 = in[(t + 0) & 63], a1 = in[(t + 1) & 63], a2 = in[(t + 2) & 63], a3 = in[(t + 3) & 63];
  float b0 = in[(t + 4) & 63], b1 = in[(t + 5) & 63], b2 = in[(t + 6) & 63], b3 = in[(t + 7) & 63];
  unsigned acc = 0;
  for (int it = 0; it < iters; ++it) {
    unsigned r;
    asm volatile(
        "{\n\t.reg .pred p<8>;\n\t"
        "setp.lt.f32 p0, %1, %5;\n\tsetp.gt.f32 p1, %1, %5;\n\t"
        "setp.lt.f32 p2, %2, %6;\n\tsetp.gt.f32 p3, %2, %6;\n\t"
        "setp.lt.f32 p4, %3, %7;\n\tsetp.gt.f32 p5, %3, %7;\n\t"
        "setp.lt.f32 p6, %4, %8;\n\tsetp.gt.f32 p7, %4, %8;\n\t"
        "setp.lt.or.f32 p0, %2, %6, p0;\n\tsetp.gt.or.f32 p1, %2, %6, p1;\n\t"
        "setp.lt.or.f32 p2, %3, %7, p2;\n\tsetp.gt.or.f32 p3, %3, %7, p3;\n\t"
        "setp.lt.or.f32 p4, %4, %8, p4;\n\tsetp.gt.or.f32 p5, %4, %8, p5;\n\t"
        "setp.lt.or.f32 p6, %1, %5, p6;\n\tsetp.gt.or.f32 p7, %1, %5, p7;\n\t"
        "setp.lt.or.f32 p0, %3, %5, p0;\n\tsetp.gt.or.f32 p1, %3, %5, p1;\n\t"
        "setp.lt.or.f32 p2, %4, %6, p2;\n\tsetp.gt.or.f32 p3, %4, %6, p3;\n\t"
        "setp.lt.or.f32 p4, %1, %7, p4;\n\tsetp.gt.or.f32 p5, %1, %7, p5;\n\t"
        "setp.lt.or.f32 p6, %2, %8, p6;\n\tsetp.gt.or.f32 p7, %2, %8, p7;\n\t"
        "setp.lt.or.f32 p0, %4, %7, p0;\n\tsetp.gt.or.f32 p1, %4, %7, p1;\n\t"
        "setp.lt.or.f32 p2, %1, %8, p2;\n\tsetp.gt.or.f32 p3, %1, %8, p3;\n\t"
        "setp.lt.or.f32 p4, %2, %5, p4;\n\tsetp.gt.or.f32 p5, %2, %5, p5;\n\t"
        "setp.lt.or.f32 p6, %3, %6, p6;\n\tsetp.gt.or.f32 p7, %3, %6, p7;\n\t"
        "setp.lt.or.f32 p0, %1, %6, p0;\n\tsetp.gt.or.f32 p1, %1, %6, p1;\n\t"
        "setp.lt.or.f32 p2, %2, %7, p2;\n\tsetp.gt.or.f32 p3, %2, %7, p3;\n\t"
        "setp.lt.or.f32 p4, %3, %8, p4;\n\tsetp.gt.or.f32 p5, %3, %8, p5;\n\t"
        "setp.lt.or.f32 p6, %4, %5, p6;\n\tsetp.gt.or.f32 p7, %4, %5, p7;\n\t"
        "setp.lt.or.f32 p0, %2, %8, p0;\n\tsetp.gt.or.f32 p1, %2, %8, p1;\n\t"
        "setp.lt.or.f32 p2, %3, %5, p2;\n\tsetp.gt.or.f32 p3, %3, %5, p3;\n\t"
        "setp.lt.or.f32 p4, %4, %6, p4;\n\tsetp.gt.or.f32 p5, %4, %6, p5;\n\t"
        "setp.lt.or.f32 p6, %1, %7, p6;\n\tsetp.gt.or.f32 p7, %1, %7, p7;\n\t"
        "setp.lt.or.f32 p0, %3, %8, p0;\n\tsetp.gt.or.f32 p1, %3, %8, p1;\n\t"
        "setp.lt.or.f32 p2, %4, %5, p2;\n\tsetp.gt.or.f32 p3, %4, %5, p3;\n\t"
        "setp.lt.or.f32 p4, %1, %6, p4;\n\tsetp.gt.or.f32 p5, %1, %6, p5;\n\t"
        "setp.lt.or.f32 p6, %2, %7, p6;\n\tsetp.gt.or.f32 p7, %2, %7, p7;\n\t"
        "setp.lt.or.f32 p0, %4, %5, p0;\n\tsetp.gt.or.f32 p1, %4, %5, p1;\n\t"
        "setp.lt.or.f32 p2, %1, %6, p2;\n\tsetp.gt.or.f32 p3, %1, %6, p3;\n\t"
        "setp.lt.or.f32 p4, %2, %7, p4;\n\tsetp.gt.or.f32 p5, %2, %7, p5;\n\t"
        "setp.lt.or.f32 p6, %3, %8, p6;\n\tsetp.gt.or.f32 p7, %3, %8, p7;\n\t"
        "xor.pred p0, p0, p1;\n\txor.pred p2, p2, p3;\n\t"
        "xor.pred p4, p4, p5;\n\txor.pred p6, p6, p7;\n\t"
        "xor.pred p0, p0, p2;\n\txor.pred p4, p4, p6;\n\txor.pred p0, p0, p4;\n\t"
        "selp.u32 %0, 1, 0, p0;\n\t}"
        : "=r"(r)
        : "f"(a0), "f"(a1), "f"(a2), "f"(a3), "f"(b0), "f"(b1), "f"(b2), "f"(b3));
    acc += r;
    // perturb one operand so the loop body cannot be hoisted (1 extra op / 64 compares)
    a0 = __uint_as_float(__float_as_uint(a0) ^ (r << 3));
  }
  if (acc == 0x7fffffffu) out[t] = acc;
}

__global__ void __launch_bounds__(256) k_peak_fp32(const float* __restrict__ in, int iters, float* out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  float x[8], y = in[t & 63], z = in[(t + 7) & 63];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = in[(t + k) & 63];
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = __fadd_rn(__fmul_rn(x[k], y), z);
  }
  float s = 0.0f;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 1234.5f) out[t] = s;
}

__global__ void __launch_bounds__(256) k_peak_smem(const float* __restrict__ in, int iters, unsigned* out) {
  __shared__ __align__(16) uint4 sbuf[2048];   // 32 KB
  for (int i = threadIdx.x; i < 2048; i += 256) sbuf[i] = make_uint4(i, i * 3, i * 5, i * 7);
  __syncthreads();
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint4 v = sbuf[(threadIdx.x + (it * 8 + u) * 256 + it) & 2047];   // a warp: 512 contiguous bytes
      acc.x ^= v.x;
      acc.y ^= v.y;
      acc.z ^= v.z;
      acc.w ^= v.w;
    }
  }
  if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x7fffffffu) out[blockIdx.x] = acc.x;
}

int launch_peak(int which, int blocks, int iters, const float* in, void* out, cudaStream_t s) {
  if (which == 2)
    k_peak_smem<<<blocks, 256, 0, s>>>(in, iters, (unsigned*)out);
  else if (which == 0)
    k_peak_fsetp<<<blocks, 256, 0, s>>>(in, iters, (unsigned*)out);
  else
    k_peak_fp32<<<blocks, 256, 0, s>>>(in, iters, (float*)out);
  MO_CHECK_LAUNCH();
  return MO_OK;
}

}  // namespace mo

extern "C" int mo_peak_issue(int32_t which, int32_t blocks, int32_t iters, const float* in64, void* out,
                             void* stream_) {
  if (which < 0 || which > 2 || blocks < 1 || iters < 1 || !in64 || !out) return MO_ERR_PARAM;
  return mo::launch_peak(which, blocks, iters, in64, out, (cudaStream_t)stream_);
}
