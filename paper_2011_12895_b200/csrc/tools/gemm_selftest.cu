// Device self-test of the tcgen05 3xTF32 GEMM against an fp64 SIMT reference on the
// same GPU (test tool; not part of the product library).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 gemm_selftest.cu ../gemm_sm100.cu
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "../gemm_i8.cuh"

using namespace tlg;

// ref[m][n] = sum_k A(m,k) B(n,k), fp64; A(m,k) = a_mn ? A[k*lda+m] : A[m*lda+k]
__global__ void ref_gemm(const float* A, long lda, bool a_mn, const float* B, long ldb, bool b_mn,
                         int M, int N, int K, double* out, double* absout) {
  int m = blockIdx.x * blockDim.x + threadIdx.x;
  int n = blockIdx.y;
  if (m >= M) return;
  double s = 0, sa = 0;
  for (int k = 0; k < K; ++k) {
    double a = a_mn ? A[long(k) * lda + m] : A[long(m) * lda + k];
    double b = b_mn ? B[long(k) * ldb + n] : B[long(n) * ldb + k];
    s += a * b;
    sa += fabs(a * b);
  }
  out[long(m) * N + n] = s;
  absout[long(m) * N + n] = sa;
}

__global__ void split_kernel(const float* x, float* hi, float* lo, long n) {
  long i = blockIdx.x * long(blockDim.x) + threadIdx.x;
  if (i < n) {
    float h = tf32_hi(x[i]);
    hi[i] = h;
    lo[i] = x[i] - h;
  }
}

struct Buf {
  float *x = nullptr, *hi = nullptr, *lo = nullptr;
  long n = 0;
  void init(long n_, std::mt19937& rng, bool binary = false) {
    n = n_;
    std::vector<float> h(n);
    std::normal_distribution<float> nd(0.f, 1.f);
    std::uniform_real_distribution<float> u(0.f, 1.f);
    for (auto& v : h) v = binary ? (u(rng) < 0.1f ? 1.f : 0.f) : nd(rng);
    TLG_CUDA(cudaMalloc(&x, n * 4));
    TLG_CUDA(cudaMalloc(&hi, n * 4));
    TLG_CUDA(cudaMalloc(&lo, n * 4));
    TLG_CUDA(cudaMemcpy(x, h.data(), n * 4, cudaMemcpyHostToDevice));
    split_kernel<<<(n + 255) / 256, 256>>>(x, hi, lo, n);
  }
};

static int failures = 0;

static bool g_fullhi = false;  // feed the full fp32 plane as "hi" (tests HW tf32 truncation)
static int g_u8 = 0;           // 1: A as uint8 planes, 2: B as uint8 planes
static int g_heads = 0;        // > 0: fused head width (fwd), timing only
static bool g_nolo = false;    // fwd/bwd: no residual output plane, timing only
static bool g_noref = false;   // timing only: skip the fp64 reference and the check

uint8_t* to_u8(const float* d, long n) {
  std::vector<float> h(n);
  std::vector<uint8_t> u(n);
  TLG_CUDA(cudaMemcpy(h.data(), d, n * 4, cudaMemcpyDeviceToHost));
  for (long i = 0; i < n; ++i) u[i] = uint8_t(h[i]);
  uint8_t* p;
  TLG_CUDA(cudaMalloc(&p, n));
  TLG_CUDA(cudaMemcpy(p, u.data(), n, cudaMemcpyHostToDevice));
  return p;
}

void check(const char* name, int M, int N, int K, bool a_mn, bool b_mn, bool a_exact, int epi,
           int splits) {
  std::mt19937 rng(M * 131 + N * 7 + K);
  Buf A, B, act, bias;
  // A stored [M][K] (K-major) or [K][M] (MN-major); same element count
  A.init(long(M) * K, rng, a_exact || g_u8 == 1);
  B.init(long(N) * K, rng, g_u8 == 2);
  act.init(long(M) * N, rng);
  bias.init(N, rng);
  // tanh'd activations in (-1,1)
  const long lda = a_mn ? M : K, ldb = b_mn ? N : K;
  double *ref, *refabs;
  TLG_CUDA(cudaMalloc(&ref, long(M) * N * 8));
  TLG_CUDA(cudaMalloc(&refabs, long(M) * N * 8));
  if (!g_noref)
    ref_gemm<<<dim3((M + 127) / 128, N), 128>>>(A.x, lda, a_mn, B.x, ldb, b_mn, M, N, K, ref,
                                                refabs);
  float *out_hi, *out_lo, *ws, *colsum;
  const int mt = std::max((M + 127) / 128, 160);  // rows: one per CTA (<= #SMs)
  TLG_CUDA(cudaMalloc(&colsum, long(mt) * N * 4));
  TLG_CUDA(cudaMemset(colsum, 0, long(mt) * N * 4));
  TLG_CUDA(cudaMalloc(&out_hi, long(M) * N * 4));
  TLG_CUDA(cudaMalloc(&out_lo, long(M) * N * 4));
  TLG_CUDA(cudaMalloc(&ws, long(splits) * M * N * 4));
  TLG_CUDA(cudaMemset(ws, 0, long(splits) * M * N * 4));
  gemm::Operand oa{g_fullhi ? A.x : A.hi, a_exact ? nullptr : A.lo, lda, a_mn};
  gemm::Operand ob{g_fullhi ? B.x : B.hi, B.lo, ldb, b_mn};
  float* expand = nullptr;
  if (g_u8 == 1) {
    oa.u8 = to_u8(A.x, long(M) * K);
  }
  if (g_u8 == 1 && !std::getenv("TLG_ST_NOEXPAND")) {
    TLG_CUDA(cudaMalloc(&expand, long(M) * K * 4));
    TLG_CUDA(cudaMemset(expand, 0xff, long(M) * K * 4));
  }
  if (g_u8 == 2) { ob.u8 = to_u8(B.x, long(N) * K); ob.lo = nullptr; }
  gemm::Params p{};
  p.out_hi = out_hi;
  p.out_lo = out_lo;
  p.ldo = N;
  p.bias = bias.x;
  // act planes: use act.x as h values (clip into (-1,1) by tanh on host side not needed)
  p.act_hi = act.x;
  p.ld_act = N;
  p.ws = ws;
  p.ws_split_stride = long(M) * N;
  p.colsum = epi == gemm::kEpiBwdTanh ? colsum : nullptr;
  p.a_expand = expand;
  float* hw = nullptr;
  if (g_heads > 0) {
    TLG_CUDA(cudaMalloc(&hw, long(N) * 8 * 4));
    TLG_CUDA(cudaMemset(hw, 0, long(N) * 8 * 4));
    TLG_CUDA(cudaMalloc(&p.head_part, long(M) * 8 * ((N + 63) / 64) * 4));
    p.head_w = hw;
    p.head_wv = hw + long(N) * 7;
    p.head_k = g_heads;
  }
  if (g_nolo) p.out_lo = nullptr;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  gemm::launch(oa, ob, M, N, K, epi, p, splits, 0);
  TLG_CUDA(cudaDeviceSynchronize());
  p.colsum = nullptr;  // timed reps below must not rewrite the checked column sums
  cudaEventRecord(e0);
  const int reps = 5;
  for (int i = 0; i < reps; ++i) gemm::launch(oa, ob, M, N, K, epi, p, splits, 0);
  cudaEventRecord(e1);
  TLG_CUDA(cudaDeviceSynchronize());
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= reps;

  std::vector<double> hr(long(M) * N), ha(long(M) * N);
  std::vector<float> hh(long(M) * N), hl(long(M) * N), hact(long(M) * N), hb(N);
  std::vector<float> hws(long(splits) * M * N);
  TLG_CUDA(cudaMemcpy(hr.data(), ref, hr.size() * 8, cudaMemcpyDeviceToHost));
  TLG_CUDA(cudaMemcpy(ha.data(), refabs, ha.size() * 8, cudaMemcpyDeviceToHost));
  TLG_CUDA(cudaMemcpy(hh.data(), out_hi, hh.size() * 4, cudaMemcpyDeviceToHost));
  TLG_CUDA(cudaMemcpy(hl.data(), out_lo, hl.size() * 4, cudaMemcpyDeviceToHost));
  TLG_CUDA(cudaMemcpy(hact.data(), act.x, hact.size() * 4, cudaMemcpyDeviceToHost));
  TLG_CUDA(cudaMemcpy(hb.data(), bias.x, hb.size() * 4, cudaMemcpyDeviceToHost));
  TLG_CUDA(cudaMemcpy(hws.data(), ws, hws.size() * 4, cudaMemcpyDeviceToHost));
  double worst = 0;
  long bad = 0;
  if (g_noref) {
    const double tf = 2.0 * M * N * K / (ms * 1e-3) / 1e12;
    printf("%-34s M=%6d N=%5d K=%6d split=%d : (timing only)  %.3f ms %.1f TF/s\n", name, M, N,
           K, splits, ms, tf);
    cudaFree(colsum); cudaFree(ref); cudaFree(refabs); cudaFree(out_hi); cudaFree(out_lo); cudaFree(ws);
    cudaFree(A.x); cudaFree(A.hi); cudaFree(A.lo); cudaFree(B.x); cudaFree(B.hi); cudaFree(B.lo);
    cudaFree(act.x); cudaFree(act.hi); cudaFree(act.lo); cudaFree(bias.x); cudaFree(bias.hi);
    cudaFree(bias.lo);
    return;
  }
  if (expand) {  // the converter's fp32 copy of the uint8 A operand must be exact
    std::vector<float> he(long(M) * K), ha(long(M) * K);
    TLG_CUDA(cudaMemcpy(he.data(), expand, he.size() * 4, cudaMemcpyDeviceToHost));
    TLG_CUDA(cudaMemcpy(ha.data(), A.x, ha.size() * 4, cudaMemcpyDeviceToHost));
    for (long i = 0; i < long(M) * K; ++i)
      if (he[i] != ha[i]) { ++bad; }
    if (bad) printf("  expanded A copy mismatches: %ld\n", bad);
    cudaFree(expand);
  }
  if (epi == gemm::kEpiBwdTanh) {
    std::vector<float> hc(long(mt) * N);
    TLG_CUDA(cudaMemcpy(hc.data(), colsum, hc.size() * 4, cudaMemcpyDeviceToHost));
    for (int n = 0; n < N; ++n) {
      double want = 0, got = 0, sa = 0;
      for (int m = 0; m < M; ++m) { want += hh[long(m) * N + n]; sa += std::fabs(hh[long(m) * N + n]); }
      for (int t = 0; t < mt; ++t) got += hc[long(t) * N + n];
      if (std::fabs(got - want) > 1e-5 * (sa + 1e-30)) ++bad;
    }
  }
  for (long i = 0; i < long(M) * N; ++i) {
    const int n = int(i % N);
    double want, got, scale;
    if (epi == gemm::kEpiStore) {
      got = 0;
      for (int s = 0; s < splits; ++s) got += hws[long(s) * M * N + i];
      want = hr[i];
      scale = ha[i] + 1e-30;
    } else if (epi == gemm::kEpiFwdTanh) {
      got = double(hh[i]);
      if (!g_nolo && std::fabs(double(hh[i]) - double(hh[i] - hl[i])) > 1e-3 * std::fabs(hh[i]) + 1e-30) got = 1e9;
      want = std::tanh(hr[i] + hb[n]);
      scale = ha[i] + 1.0;
    } else {
      const double h = hact[i];
      got = double(hh[i]);
      want = hr[i] * (1 - h * h);
      scale = (ha[i] + 1e-30) * std::max(1.0, std::fabs(1 - h * h));
    }
    const double err = std::fabs(got - want) / scale;
    if (!(err <= (K > 20000 ? 1e-5 : 2e-6))) ++bad;
    if (!(err <= worst)) worst = std::isfinite(err) ? std::max(worst, err) : 1e30;
  }
  const double tflops = 2.0 * M * N * K / (ms * 1e-3) / 1e12;
  printf("%-34s M=%6d N=%5d K=%6d split=%d : worst rel %.3e bad %ld  %.3f ms %.1f TF/s  %s\n",
         name, M, N, K, splits, worst, bad, ms, tflops, bad ? "FAIL" : "ok");
  if (bad) ++failures;
  cudaFree(colsum); cudaFree(ref); cudaFree(refabs); cudaFree(out_hi); cudaFree(out_lo); cudaFree(ws);
  cudaFree(A.x); cudaFree(A.hi); cudaFree(A.lo); cudaFree(B.x); cudaFree(B.hi); cudaFree(B.lo);
  cudaFree(act.x); cudaFree(act.hi); cudaFree(act.lo); cudaFree(bias.x); cudaFree(bias.hi);
  cudaFree(bias.lo);
}

// Binary planes (bit-packed) x fixed-point int8 pieces of W (kind::i8), fused bias + tanh.
static bool g_i8_nolo = false;  // the consumers derive the residual: no out_lo plane

void check_i8(const char* name, int M, int N, int K) {
  std::mt19937 rng(M * 17 + N * 3 + K);
  Buf A, B, bias;
  A.init(long(M) * K, rng, true);
  B.init(long(N) * K, rng);
  bias.init(N, rng);
  double *ref, *refabs;
  TLG_CUDA(cudaMalloc(&ref, long(M) * N * 8));
  TLG_CUDA(cudaMalloc(&refabs, long(M) * N * 8));
  ref_gemm<<<dim3((M + 127) / 128, N), 128>>>(A.x, K, false, B.x, K, false, M, N, K, ref, refabs);
  const long rowb = ((K + 7) / 8 + 15) / 16 * 16, Kp = (K + 15) / 16 * 16;
  std::vector<float> ha(long(M) * K);
  TLG_CUDA(cudaMemcpy(ha.data(), A.x, ha.size() * 4, cudaMemcpyDeviceToHost));
  std::vector<uint8_t> hb(long(M) * rowb, 0);
  for (long m = 0; m < M; ++m)
    for (long k = 0; k < K; ++k)
      if (ha[m * K + k] != 0.f) hb[m * rowb + k / 8] |= uint8_t(1u << (k % 8));
  uint8_t* bits;
  int8_t* q;
  float *scale, *out, *out_lo;
  TLG_CUDA(cudaMalloc(&bits, hb.size()));
  TLG_CUDA(cudaMemcpy(bits, hb.data(), hb.size(), cudaMemcpyHostToDevice));
  TLG_CUDA(cudaMalloc(&q, 3 * long(N) * Kp));
  TLG_CUDA(cudaMalloc(&scale, N * 4));
  TLG_CUDA(cudaMalloc(&out, long(M) * N * 4));
  TLG_CUDA(cudaMalloc(&out_lo, long(M) * N * 4));
  gemm::launch_quantize_rows(B.x, N, K, K, q, Kp, scale, 0);
  float* lo_arg = g_i8_nolo ? nullptr : out_lo;
  gemm::launch_i8_bits_fwd(bits, rowb, q, Kp, scale, bias.x, M, N, K, out, lo_arg, N, 0);
  TLG_CUDA(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  const int reps = 5;
  for (int i = 0; i < reps; ++i)
    gemm::launch_i8_bits_fwd(bits, rowb, q, Kp, scale, bias.x, M, N, K, out, lo_arg, N, 0);
  cudaEventRecord(e1);
  TLG_CUDA(cudaDeviceSynchronize());
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= reps;
  std::vector<double> hr(long(M) * N), hab(long(M) * N);
  std::vector<float> hh(long(M) * N), hl(long(M) * N), hbias(N);
  TLG_CUDA(cudaMemcpy(hr.data(), ref, hr.size() * 8, cudaMemcpyDeviceToHost));
  TLG_CUDA(cudaMemcpy(hab.data(), refabs, hab.size() * 8, cudaMemcpyDeviceToHost));
  TLG_CUDA(cudaMemcpy(hh.data(), out, hh.size() * 4, cudaMemcpyDeviceToHost));
  TLG_CUDA(cudaMemcpy(hl.data(), out_lo, hl.size() * 4, cudaMemcpyDeviceToHost));
  TLG_CUDA(cudaMemcpy(hbias.data(), bias.x, N * 4, cudaMemcpyDeviceToHost));
  double worst = 0;
  long bad = 0;
  for (long i = 0; i < long(M) * N; ++i) {
    const int n = int(i % N);
    double got = hh[i];
    uint32_t u;
    std::memcpy(&u, &hh[i], 4);
    u &= 0xFFFFE000u;
    float th;
    std::memcpy(&th, &u, 4);
    if (!g_i8_nolo && hl[i] != hh[i] - th) got = 1e9;  // residual plane = x - trunc_tf32(x)
    const double want = std::tanh(hr[i] + hbias[n]);
    const double err = std::fabs(got - want) / (hab[i] + 1.0);
    if (!(err <= 2e-6)) ++bad;
    if (!(err <= worst)) worst = std::isfinite(err) ? std::max(worst, err) : 1e30;
  }
  const double tflops = 2.0 * M * N * K / (ms * 1e-3) / 1e12;
  printf("%-34s M=%6d N=%5d K=%6d split=1 : worst rel %.3e bad %ld  %.3f ms %.1f TF/s  %s\n",
         name, M, N, K, worst, bad, ms, tflops, bad ? "FAIL" : "ok");
  if (bad) ++failures;
  cudaFree(ref); cudaFree(refabs); cudaFree(bits); cudaFree(q); cudaFree(scale); cudaFree(out);
  cudaFree(out_lo); cudaFree(A.x); cudaFree(A.hi); cudaFree(A.lo); cudaFree(B.x); cudaFree(B.hi);
  cudaFree(B.lo); cudaFree(bias.x); cudaFree(bias.hi); cudaFree(bias.lo);
}

// dW = dZ^T X with X bit-packed binary planes and dZ as per-split fixed-point pieces.
void check_i8_dw(const char* name, int M, int N, int K, int kb_per_split) {
  std::mt19937 rng(M * 5 + N * 11 + K);
  Buf Z, X;
  Z.init(long(K) * M, rng);        // dZ stored [K=frames][M]
  X.init(long(K) * N, rng, true);  // planes stored [K][N]
  double *ref, *refabs;
  TLG_CUDA(cudaMalloc(&ref, long(M) * N * 8));
  TLG_CUDA(cudaMalloc(&refabs, long(M) * N * 8));
  ref_gemm<<<dim3((M + 127) / 128, N), 128>>>(Z.x, M, true, X.x, N, true, M, N, K, ref, refabs);
  const long rowb = ((N + 7) / 8 + 15) / 16 * 16;
  const int rows_split = kb_per_split * 128;
  const int splits = (K + rows_split - 1) / rows_split;
  std::vector<float> hz(long(K) * M), hx(long(K) * N);
  TLG_CUDA(cudaMemcpy(hz.data(), Z.x, hz.size() * 4, cudaMemcpyDeviceToHost));
  TLG_CUDA(cudaMemcpy(hx.data(), X.x, hx.size() * 4, cudaMemcpyDeviceToHost));
  std::vector<uint8_t> hb(long(K) * rowb, 0);
  for (long f = 0; f < K; ++f)
    for (long n = 0; n < N; ++n)
      if (hx[f * N + n] != 0.f) hb[f * rowb + n / 8] |= uint8_t(1u << (n % 8));
  std::vector<float> cm(long(splits) * M, 0.f);
  for (long f = 0; f < K; ++f)
    for (int m = 0; m < M; ++m) {
      float& c = cm[(f / rows_split) * M + m];
      c = std::max(c, std::fabs(hz[f * M + m]));
    }
  uint8_t* bits;
  int8_t* P;
  unsigned* colmax;
  float* ws;
  TLG_CUDA(cudaMalloc(&bits, hb.size()));
  TLG_CUDA(cudaMemcpy(bits, hb.data(), hb.size(), cudaMemcpyHostToDevice));
  TLG_CUDA(cudaMalloc(&colmax, cm.size() * 4));
  TLG_CUDA(cudaMemcpy(colmax, cm.data(), cm.size() * 4, cudaMemcpyHostToDevice));
  TLG_CUDA(cudaMalloc(&P, 3L * K * M));
  TLG_CUDA(cudaMalloc(&ws, long(splits) * M * N * 4));
  gemm::launch_quantize_cols(Z.x, K, M, M, colmax, rows_split, P, 0);
  gemm::launch_i8_bits_dw(P, bits, rowb, colmax, M, N, K, kb_per_split, ws, 0);
  TLG_CUDA(cudaDeviceSynchronize());
  cudaEvent_t e0, e1, e2;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventCreate(&e2);
  const int reps = 5;
  cudaEventRecord(e0);
  for (int i = 0; i < reps; ++i) gemm::launch_quantize_cols(Z.x, K, M, M, colmax, rows_split, P, 0);
  cudaEventRecord(e1);
  for (int i = 0; i < reps; ++i)
    gemm::launch_i8_bits_dw(P, bits, rowb, colmax, M, N, K, kb_per_split, ws, 0);
  cudaEventRecord(e2);
  TLG_CUDA(cudaDeviceSynchronize());
  float msq = 0, ms = 0;
  cudaEventElapsedTime(&msq, e0, e1);
  cudaEventElapsedTime(&ms, e1, e2);
  msq /= reps;
  ms /= reps;
  std::vector<double> hr(long(M) * N), ha(long(M) * N);
  std::vector<float> hw(long(splits) * M * N);
  TLG_CUDA(cudaMemcpy(hr.data(), ref, hr.size() * 8, cudaMemcpyDeviceToHost));
  TLG_CUDA(cudaMemcpy(ha.data(), refabs, ha.size() * 8, cudaMemcpyDeviceToHost));
  TLG_CUDA(cudaMemcpy(hw.data(), ws, hw.size() * 4, cudaMemcpyDeviceToHost));
  double worst = 0;
  long bad = 0;
  for (long i = 0; i < long(M) * N; ++i) {
    double got = 0;
    for (int sp = 0; sp < splits; ++sp) got += hw[long(sp) * M * N + i];
    const double err = std::fabs(got - hr[i]) / (ha[i] + 1e-30);
    if (!(err <= 2e-6)) ++bad;
    if (!(err <= worst)) worst = std::isfinite(err) ? std::max(worst, err) : 1e30;
  }
  const double tflops = 2.0 * M * N * K / (ms * 1e-3) / 1e12;
  printf("%-34s M=%6d N=%5d K=%6d split=%d : worst rel %.3e bad %ld  %.3f ms %.1f TF/s (quantize %.3f ms)  %s\n",
         name, M, N, K, splits, worst, bad, ms, tflops, msq, bad ? "FAIL" : "ok");
  if (bad) ++failures;
  cudaFree(ref); cudaFree(refabs); cudaFree(bits); cudaFree(P); cudaFree(colmax); cudaFree(ws);
  cudaFree(Z.x); cudaFree(Z.hi); cudaFree(Z.lo); cudaFree(X.x); cudaFree(X.hi); cudaFree(X.lo);
}

// tanh activations as int8 pieces (scale 1/127) x int8 weight pieces (kind::i8, 6 MMAs)
static void host_act_pieces(const std::vector<float>& o, long M, long K, std::vector<int8_t>& q) {
  const float kMagic = 12582912.f;
  q.assign(3 * M * K, 0);
  for (long i = 0; i < M * K; ++i) {
    volatile float x = o[i] * 127.f;
    volatile float m0 = x + kMagic;
    volatile float r0 = m0 - kMagic;
    volatile float x1 = (x - r0) * 128.f;
    volatile float m1 = x1 + kMagic;
    volatile float r1 = m1 - kMagic;
    volatile float x2 = (x1 - r1) * 128.f;
    volatile float m2 = x2 + kMagic;
    float f0 = m0, f1 = m1, f2 = m2;
    uint32_t u0, u1, u2;
    std::memcpy(&u0, &f0, 4); std::memcpy(&u1, &f1, 4); std::memcpy(&u2, &f2, 4);
    q[i] = int8_t(u0 & 0xFF);
    q[M * K + i] = int8_t(u1 & 0xFF);
    q[2 * M * K + i] = int8_t(u2 & 0xFF);
  }
}

void check_i8x2(const char* name, int M, int N, int K) {
  std::mt19937 rng(M * 3 + N * 7 + K);
  std::uniform_real_distribution<float> u(-0.999f, 0.999f);
  std::vector<float> ha(long(M) * K);
  for (auto& v : ha) v = u(rng);
  float* A;
  TLG_CUDA(cudaMalloc(&A, ha.size() * 4));
  TLG_CUDA(cudaMemcpy(A, ha.data(), ha.size() * 4, cudaMemcpyHostToDevice));
  Buf B, bias;
  B.init(long(N) * K, rng);
  bias.init(N, rng);
  double *ref, *refabs;
  TLG_CUDA(cudaMalloc(&ref, long(M) * N * 8));
  TLG_CUDA(cudaMalloc(&refabs, long(M) * N * 8));
  ref_gemm<<<dim3((M + 127) / 128, N), 128>>>(A, K, false, B.x, K, false, M, N, K, ref, refabs);
  std::vector<int8_t> hq;
  host_act_pieces(ha, M, K, hq);
  int8_t *aq, *wq;
  float *scale, *out, *out_lo;
  const long Kp = (K + 15) / 16 * 16;
  TLG_CUDA(cudaMalloc(&aq, hq.size()));
  TLG_CUDA(cudaMemcpy(aq, hq.data(), hq.size(), cudaMemcpyHostToDevice));
  TLG_CUDA(cudaMalloc(&wq, 3 * long(N) * Kp));
  TLG_CUDA(cudaMalloc(&scale, N * 4));
  TLG_CUDA(cudaMalloc(&out, long(M) * N * 4));
  TLG_CUDA(cudaMalloc(&out_lo, long(M) * N * 4));
  gemm::launch_quantize_rows(B.x, N, K, K, wq, Kp, scale, 0);
  auto run = [&] {
    gemm::launch_i8x2_fwd(aq, wq, Kp, scale, bias.x, M, N, K, out, out_lo, N, nullptr, nullptr, 0,
                          nullptr, 0);
  };
  run();
  TLG_CUDA(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int i = 0; i < 5; ++i) run();
  cudaEventRecord(e1);
  TLG_CUDA(cudaDeviceSynchronize());
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= 5;
  std::vector<double> hr(long(M) * N), hab(long(M) * N);
  std::vector<float> hh(long(M) * N), hl(long(M) * N), hbias(N);
  TLG_CUDA(cudaMemcpy(hr.data(), ref, hr.size() * 8, cudaMemcpyDeviceToHost));
  TLG_CUDA(cudaMemcpy(hab.data(), refabs, hab.size() * 8, cudaMemcpyDeviceToHost));
  TLG_CUDA(cudaMemcpy(hh.data(), out, hh.size() * 4, cudaMemcpyDeviceToHost));
  TLG_CUDA(cudaMemcpy(hl.data(), out_lo, hl.size() * 4, cudaMemcpyDeviceToHost));
  TLG_CUDA(cudaMemcpy(hbias.data(), bias.x, N * 4, cudaMemcpyDeviceToHost));
  double worst = 0;
  long bad = 0;
  for (long i = 0; i < long(M) * N; ++i) {
    const int n = int(i % N);
    double got = hh[i];
    uint32_t bits;
    std::memcpy(&bits, &hh[i], 4);
    bits &= 0xFFFFE000u;
    float th;
    std::memcpy(&th, &bits, 4);
    if (hl[i] != hh[i] - th) got = 1e9;
    const double want = std::tanh(hr[i] + hbias[n]);
    const double err = std::fabs(got - want) / (hab[i] + 1.0);
    if (!(err <= 2e-6)) ++bad;
    if (!(err <= worst)) worst = std::isfinite(err) ? std::max(worst, err) : 1e30;
  }
  const double tflops = 2.0 * M * N * K / (ms * 1e-3) / 1e12;
  printf("%-34s M=%6d N=%5d K=%6d split=1 : worst rel %.3e bad %ld  %.3f ms %.1f TF/s  %s\n",
         name, M, N, K, worst, bad, ms, tflops, bad ? "FAIL" : "ok");
  if (bad) ++failures;
  cudaFree(A); cudaFree(ref); cudaFree(refabs); cudaFree(aq); cudaFree(wq); cudaFree(scale);
  cudaFree(out); cudaFree(out_lo); cudaFree(B.x); cudaFree(B.hi); cudaFree(B.lo); cudaFree(bias.x);
  cudaFree(bias.hi); cudaFree(bias.lo);
}

// Derived lo planes (Operand::lo_smem): the GEMM computes lo = x - trunc_tf32(x) in shared
// memory; the result must equal, bit for bit, the same GEMM fed the residual planes from
// HBM, and must not vary across repeats.
void check_lod(const char* name, int M, int N, int K, bool a_mn, bool b_mn, int epi, int splits,
               int lod) {
  std::mt19937 rng(M * 31 + N * 17 + K + lod);
  Buf A, B, act, bias;
  A.init(long(M) * K, rng);
  B.init(long(N) * K, rng);
  act.init(long(M) * N, rng);
  bias.init(N, rng);
  const long lda = a_mn ? M : K, ldb = b_mn ? N : K;
  const long outn = epi == gemm::kEpiStore ? long(splits) * M * N : long(M) * N;
  float* outs[7];
  for (auto& o : outs) {
    TLG_CUDA(cudaMalloc(&o, outn * 4));
    TLG_CUDA(cudaMemset(o, 0, outn * 4));
  }
  auto run = [&](bool derive, float* out) {
    gemm::Operand oa{A.x, A.lo, lda, a_mn};
    gemm::Operand ob{B.x, B.lo, ldb, b_mn};
    if (derive && (lod & 1)) { oa.lo = nullptr; oa.lo_smem = true; }
    if (derive && (lod & 2)) { ob.lo = nullptr; ob.lo_smem = true; }
    gemm::Params p{};
    p.out_hi = out;
    p.ldo = N;
    p.bias = bias.x;
    p.act_hi = act.x;
    p.ld_act = N;
    p.ws = out;
    p.ws_split_stride = long(M) * N;
    gemm::launch(oa, ob, M, N, K, epi, p, splits, 0);
  };
  run(false, outs[0]);
  for (int r = 1; r < 7; ++r) run(true, outs[r]);
  TLG_CUDA(cudaDeviceSynchronize());
  std::vector<float> ref(outn), got(outn);
  TLG_CUDA(cudaMemcpy(ref.data(), outs[0], outn * 4, cudaMemcpyDeviceToHost));
  long bad = 0;
  for (int r = 1; r < 7; ++r) {
    TLG_CUDA(cudaMemcpy(got.data(), outs[r], outn * 4, cudaMemcpyDeviceToHost));
    for (long i = 0; i < outn; ++i)
      if (std::memcmp(&ref[i], &got[i], 4) != 0) ++bad;
  }
  printf("%-34s M=%6d N=%5d K=%6d split=%d lod=%d : %s (%ld mismatching words over 6 runs)\n",
         name, M, N, K, splits, lod, bad ? "FAIL" : "ok", bad);
  if (bad) ++failures;
  for (auto& o : outs) cudaFree(o);
}

int main(int argc, char** argv) {
  try {
    using namespace gemm;
    check("fwd tanh K/K", 300, 256, 200, false, false, false, kEpiFwdTanh, 1);
    check("fwd tanh K/K exactA", 300, 256, 200, false, false, true, kEpiFwdTanh, 1);
    check("fwd tanh K/K N=100", 257, 100, 96, false, false, false, kEpiFwdTanh, 1);
    check("fwd tanh K/K N=64", 128, 64, 64, false, false, false, kEpiFwdTanh, 1);
    check("dX bwd K/MN", 300, 256, 256, false, true, false, kEpiBwdTanh, 1);
    check("dX bwd K/MN N=64", 200, 64, 256, false, true, false, kEpiBwdTanh, 1);
    check("dX bwd K/K", 300, 256, 256, false, false, false, kEpiBwdTanh, 1);
    check("dW store MN/MN", 256, 200, 1000, true, true, false, kEpiStore, 1);
    check("dW store MN/MN split4", 256, 200, 1000, true, true, false, kEpiStore, 4);
    check("dW store MN/MN exactB", 256, 1936, 2048, true, true, false, kEpiStore, 2);
    check("store K/K", 256, 256, 512, false, false, false, kEpiStore, 1);
    check_lod("LOD fwd tanh K/K", 300, 256, 200, false, false, kEpiFwdTanh, 1, 1);
    check_lod("LOD fwd tanh K/K pair", 4096, 256, 512, false, false, kEpiFwdTanh, 1, 1);
    // 128-column tiles (short K): two epilogue warp groups on alternate chunks
    check_lod("LOD fwd tanh K/K pair short-K", 4096, 256, 256, false, false, kEpiFwdTanh, 1, 1);
    check_lod("LOD fwd tanh K/K short-K N=1024", 1000, 1024, 64, false, false, kEpiFwdTanh, 1, 1);
    check_lod("LOD dX bwd K/MN", 300, 256, 256, false, true, kEpiBwdTanh, 1, 1);
    check_lod("LOD dX bwd K/MN pair", 20480, 512, 512, false, true, kEpiBwdTanh, 1, 1);
    check_lod("LOD dX bwd K/MN pair short-K", 20480, 256, 256, false, true, kEpiBwdTanh, 1, 1);
    check_lod("LOD dW store MN/MN", 256, 200, 1000, true, true, kEpiStore, 1, 3);
    check_lod("LOD dW store MN/MN split4", 512, 512, 20480, true, true, kEpiStore, 4, 3);
    check_lod("LOD dW store MN/MN split1 pair", 512, 512, 20480, true, true, kEpiStore, 1, 3);
    g_fullhi = true;
    check("FULLHI fwd tanh K/K", 300, 256, 200, false, false, false, kEpiFwdTanh, 1);
    check("FULLHI dX bwd K/MN", 300, 256, 256, false, true, false, kEpiBwdTanh, 1);
    check("FULLHI dW store MN/MN", 256, 200, 1000, true, true, false, kEpiStore, 1);
    g_fullhi = false;
    g_u8 = 1;
    check("U8A fwd tanh K/K", 300, 256, 208, false, false, true, kEpiFwdTanh, 1);
    check("U8A fwd tanh K/K N=100", 257, 100, 1936, false, false, true, kEpiFwdTanh, 1);
    g_u8 = 2;
    check("U8B dW store MN/MN", 256, 1936, 1000, true, true, false, kEpiStore, 3);
    check("U8B dW store MN/MN N=64", 200, 64, 300, true, true, false, kEpiStore, 1);
    g_u8 = 0;
    check_i8("I8 bits fwd", 300, 256, 200);
    check_i8("I8 bits fwd N=100 K=1936", 700, 100, 1936);
    check_i8("I8 bits fwd pair", 4096, 256, 1936);
    g_i8_nolo = true;  // decoupled-ring kernel (no residual plane)
    check_i8("I8 bits fwd pair no-lo", 4096, 256, 1936);
    check_i8("I8 bits fwd pair no-lo ragged", 700, 200, 1000);
    check_i8("I8 bits fwd pair no-lo ragged pairs", 20000, 200, 1000);  // 256-col tiles
    check_i8("I8 bits fwd pair no-lo C3", 131072, 256, 1936);
    g_i8_nolo = false;
    check_i8x2("I8x2 fwd", 512, 256, 256);
    check_i8x2("I8x2 fwd ragged", 700, 200, 96);
    check_i8_dw("I8 bits dW", 128, 200, 1000, 2);
    check_i8_dw("I8 bits dW pair", 256, 1936, 4096, 8);
    check_i8_dw("I8 bits dW ragged", 256, 300, 1300, 4);
    if (argc > 1 && std::string(argv[1]) == "i8") {
      check_i8("perf I8 bits fwd C3 L1", 131072, 256, 1936);
      g_i8_nolo = true;
      check_i8("perf I8 bits fwd C3 L1 no-lo", 131072, 256, 1936);
      check_i8("perf I8 bits fwd C3 L1 no-lo", 131072, 256, 1936);
      g_i8_nolo = false;
    } else if (argc > 1 && std::string(argv[1]) == "c5") {
      g_noref = true;  // C5 trunk shapes (4x2048, 131,072 frames per shard)
      check("perf fwd C5", 131072, 2048, 2048, false, false, false, kEpiFwdTanh, 1);
      check("perf dX C5 K/MN", 131072, 2048, 2048, false, true, false, kEpiBwdTanh, 1);
      check("perf dX C5 K/K", 131072, 2048, 2048, false, false, false, kEpiBwdTanh, 1);
      for (int sp : {1, 2, 4, 8, 15, 37})
        check("perf dW C5", 2048, 2048, 131072, true, true, false, kEpiStore, sp);
      g_noref = false;
    } else if (argc > 1) {
      check_i8("perf I8 bits fwd C3 L1", 131072, 256, 1936);
      check_i8_dw("perf I8 bits dW C3 L1", 256, 1936, 131072, 114);
      check_i8x2("perf I8x2 fwd C3 L2", 131072, 256, 256);
      g_u8 = 1;
      check("perf U8 fwd C3 L1", 131072, 256, 1936, false, false, true, kEpiFwdTanh, 1);
      g_u8 = 2;
      check("perf U8 dW C3 L1", 256, 1936, 131072, true, true, false, kEpiStore, 9);
      g_u8 = 0;
      // throughput shapes (C3 layer 1 forward, C5 layer forward)
      check("perf fwd C3 L1", 131072, 256, 1936, false, false, true, kEpiFwdTanh, 1);
      check("perf fwd C5", 131072, 2048, 2048, false, false, false, kEpiFwdTanh, 1);
      check("perf dW C3 L1", 256, 1936, 131072, true, true, false, kEpiStore, 9);
      check("perf dW C3 L2", 256, 256, 131072, true, true, false, kEpiStore, 74);
      check("perf dX C3 L2", 131072, 256, 256, false, true, false, kEpiBwdTanh, 1);
      check("perf fwd C3 L2", 131072, 256, 256, false, false, false, kEpiFwdTanh, 1);
      check("perf fwd C4 L2", 65536, 1024, 1024, false, false, false, kEpiFwdTanh, 1);
      g_nolo = true;
      check("perf fwd C3 L2 no-lo", 131072, 256, 256, false, false, false, kEpiFwdTanh, 1);
      g_heads = 7;
      check("perf fwd C3 L2 heads no-lo", 131072, 256, 256, false, false, false, kEpiFwdTanh, 1);
      g_heads = 0;
      g_nolo = false;
    }
  } catch (const std::exception& e) {
    printf("EXCEPTION: %s\n", e.what());
    return 2;
  }
  printf("%s\n", failures ? "GEMM SELFTEST FAILED" : "GEMM SELFTEST PASSED");
  return failures ? 1 : 0;
}
