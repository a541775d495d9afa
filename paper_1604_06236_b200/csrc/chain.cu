// chain.cu — fused FFT chains of the type-4 / type-5 solves, one signal per
// tile row (signal-major; batches of 16 or more use chain_bm.cu).
//
// With P = PR*PC (PR = PC = M for even powers of two, PR = 2 PC for odd
// ones), the P-point vectors in the layout p = k + PR m, the fine grid
// n = 2P split PR x 2PC and K = P/2 = PR (PC/2), the four-step FFT
// decompositions of FFT_2P, IFFT_P, FFT_P and IFFT_2P can be chosen so that
// the row pass of one transform produces exactly the columns the next
// transform's column pass needs (the band (p - K) mod n of FFT_2P row k is
// column k of the P layout because K = 0 mod PR).  Each kernel below
// therefore does  row FFT -> elementwise stage -> column FFT  on CT rows of
// one signal entirely in shared memory, so every fused stage costs one HBM
// read and one HBM write instead of two of each:
//
//   type 5:  spread -> colFFT_2P -> [rowFFT_2P | band*deconv*decay | colIFFT_P]
//            -> [rowIFFT_P | *ks | colFFT_P] -> [rowFFT_P | *coef]
//   type 4:  [colIFFT_P *decay] -> [rowIFFT_P | *ks | colFFT_P]
//            -> [rowFFT_P | *coef*deconv, pad | colIFFT_2P] -> rowIFFT_2P -> gather
//
// (reference: inverse.py:101-143, forward.py:26-102, 133-162).
#include "fft_fast.cuh"
#include "ops.cuh"

namespace nfft45 {

namespace {

__device__ __forceinline__ double2 rscale(double2 v, double s) { return make_double2(v.x * s, v.y * s); }


}  // namespace

// K3: rows k1 < PR of the FFT_2P pass-A output (length 2PC) -> band select
// p = k1 + PR m1 (m1 < PC) with (X deconv [- sub]) decay -> column IFFT_P
// (length PC) -> twiddle W_P^{+k1 m} -> U[m PR + k1].
template <int PR, int PC, int C>
__global__ void __launch_bounds__(fast_threads<2 * PC, C>(), 2) kc_band(
    const double2* __restrict__ T, double2* __restrict__ U, const double2* __restrict__ twR,
    const double2* __restrict__ twC, const double2* __restrict__ loP, const double2* __restrict__ hiP, int sP,
    const double* __restrict__ deconv, const double* __restrict__ decay, const double* __restrict__ dd,
    const double2* __restrict__ sub, const double2* __restrict__ twQ, int Q, double2* __restrict__ rsave) {
  pdl_enter();  // programmatic dependent launch: wait for the producer grid
  constexpr int64_t P = (int64_t)PR * PC, n = 2 * P;
  constexpr int NR = 2 * PC;
  extern __shared__ double2 sm[];
  const int r0 = blockIdx.x * C;
  const int64_t bi = blockIdx.y;
  const double2* Tin = T + bi * n;
  auto ld1 = [&](int i, int c) -> double2 { return Tin[(int64_t)(r0 + c) * NR + i]; };
  auto st1 = [&](int k2, int c, double2 v) {
    const int m1 = (k2 + PC / 2) & (NR - 1);  // (k2 + K/PR) mod 2PC, K/PR = PC/2
    if (m1 < PC) {
      const int64_t p = (int64_t)(r0 + c) + (int64_t)PR * m1;
      if (sub) {  // type-4 residual: (X deconv - A) decay
        v = rscale(v, __ldg(&deconv[p]));
        v = csub(v, sub[bi * P + p]);
        if (rsave) rsave[bi * P + p] = v;  // the residual itself (norms for passes >= 2)
        v = rscale(v, __ldg(&decay[p]));
      } else {
        v = rscale(v, __ldg(&dd[p]));  // deconv * decay
      }
      sm[sidx<PC, C, true>(m1, c)] = v;
    }
  };
  fast_tile_fft<NR, C, -1, true>(sm, ld1, st1, twR);
  __syncthreads();
  auto ld2 = [&](int i, int c) -> double2 { return sm[sidx<PC, C, true>(i, c)]; };
  auto st2 = [&](int k1, int c, double2 v) { U[bi * P + (int64_t)k1 * PR + r0 + c] = v; };
  const FourStepTw<+1> pt{loP, hiP, sP, twQ, Q, r0, -1};
  fast_tile_fft_smem<PC, C, +1, true, HalfTr<PC>>(sm, ld2, st2, twC, pt);
}

// K4 / K2': rows r < PC of U (length PR) -> row IFFT_P -> * ks[r + PC k2] ->
// column FFT_P (length PR, column r of the layout q = r + PC k2) -> twiddle
// W_P^{-r k} -> Z[k PC + r].
template <int PR, int PC, int C>
__global__ void __launch_bounds__(fast_threads<PR, C>()) kc_mid(const double2* __restrict__ U, double2* __restrict__ Z,
                                                               const double2* __restrict__ tw,
                                                               const double2* __restrict__ loP,
                                                               const double2* __restrict__ hiP, int sP,
                                                               const double2* __restrict__ ks,
                                                               const double2* __restrict__ twQ, int Q) {
  pdl_enter();  // programmatic dependent launch: wait for the producer grid
  constexpr int64_t P = (int64_t)PR * PC;
  extern __shared__ double2 sm[];
  const int r0 = blockIdx.x * C;
  const int64_t bi = blockIdx.y;
  const double2* Uin = U + bi * P;
  auto ld1 = [&](int i, int c) -> double2 { return Uin[(int64_t)(r0 + c) * PR + i]; };
  auto st1 = [&](int k2, int c, double2 v) {
    const int64_t p = (int64_t)(r0 + c) + (int64_t)PC * k2;
    sm[sidx<PR, C, true>(k2, c)] = cmul(v, __ldg(&ks[p]));
  };
  fast_tile_fft<PR, C, +1, true>(sm, ld1, st1, tw);
  __syncthreads();
  auto ld2 = [&](int i, int c) -> double2 { return sm[sidx<PR, C, true>(i, c)]; };
  auto st2 = [&](int k1, int c, double2 v) { Z[bi * P + (int64_t)k1 * PC + r0 + c] = v; };
  const FourStepTw<-1> pt{loP, hiP, sP, twQ, Q, r0, -1};
  fast_tile_fft_smem<PR, C, -1, true>(sm, ld2, st2, tw, pt);
}

// K3' / K5+: rows r < PR of Z (length PC) -> row FFT_P -> S_p * coef_p
// (p = r + PR k2); optional x = xsub - S (refinement) stored to xout; then
// * deconv_p, zero-padded into the IFFT_2P column (length 2PC) at
// n1 = (k2 - PC/2) mod 2PC -> column IFFT -> twiddle W_n^{+r t} -> Y[t PR + r].
template <int PR, int PC, int C>
__global__ void __launch_bounds__(fast_threads<2 * PC, C>(), 2) kc_pad(
    const double2* __restrict__ Z, double2* __restrict__ Y, const double2* __restrict__ twR,
    const double2* __restrict__ twC, const double2* __restrict__ loN, const double2* __restrict__ hiN, int sN,
    const double* __restrict__ coef, const double* __restrict__ deconv, const double* __restrict__ cd,
    const double2* __restrict__ xsub, double2* __restrict__ xout, const double2* __restrict__ twQ, int Q) {
  pdl_enter();  // programmatic dependent launch: wait for the producer grid
  constexpr int64_t P = (int64_t)PR * PC, n = 2 * P;
  constexpr int NC = 2 * PC;
  extern __shared__ double2 sm[];
  const int r0 = blockIdx.x * C;
  const int64_t bi = blockIdx.y;
  const double2* Zin = Z + bi * P;
  auto ld1 = [&](int i, int c) -> double2 { return Zin[(int64_t)(r0 + c) * PC + i]; };
  auto st1 = [&](int k2, int c, double2 v) {
    const int64_t p = (int64_t)(r0 + c) + (int64_t)PR * k2;
    if (xout) {  // refinement: x = (xsub -) S coef is stored, then deconvolved
      v = rscale(v, __ldg(&coef[p]));
      if (xsub) v = csub(xsub[bi * P + p], v);
      xout[bi * P + p] = v;
      v = rscale(v, __ldg(&deconv[p]));
    } else {
      v = rscale(v, __ldg(&cd[p]));  // coef * deconv
    }
    const int n1 = (k2 - PC / 2) & (NC - 1);
    sm[sidx<NC, C, true>(n1, c)] = v;
    sm[sidx<NC, C, true>((n1 + PC) & (NC - 1), c)] = make_double2(0.0, 0.0);
  };
  fast_tile_fft<PC, C, -1, true, HalfTr<PC>>(sm, ld1, st1, twR);
  __syncthreads();
  auto ld2 = [&](int i, int c) -> double2 { return sm[sidx<NC, C, true>(i, c)]; };
  auto st2 = [&](int k1, int c, double2 v) { Y[bi * n + (int64_t)k1 * PR + r0 + c] = v; };
  const FourStepTw<+1> pt{loN, hiN, sN, twQ, Q, r0, -1};
  fast_tile_fft_smem<NC, C, +1, true>(sm, ld2, st2, twC, pt);
}

// K5 / K4': rows of length L (row pass), output index k1 + R1 k2 with
// optional real post-table and optional out = xsub - v.
template <int L, int C, int S>
__global__ void __launch_bounds__(fast_threads<L, C>()) kc_row(const double2* __restrict__ in,
                                                              double2* __restrict__ out, int64_t len, int64_t R1,
                                                              const double2* __restrict__ tw,
                                                              const double* __restrict__ post,
                                                              const double2* __restrict__ xsub) {
  pdl_enter();  // programmatic dependent launch: wait for the producer grid
  extern __shared__ double2 sm[];
  const int r0 = blockIdx.x * C;
  const int64_t base = (int64_t)blockIdx.y * len;
  auto ld = [&](int i, int c) -> double2 { return in[base + (int64_t)(r0 + c) * L + i]; };
  auto st = [&](int k2, int c, double2 v) {
    const int64_t idx = (int64_t)(r0 + c) + R1 * k2;
    if (post) v = rscale(v, __ldg(&post[idx]));
    if (xsub) v = csub(xsub[base + idx], v);
    out[base + idx] = v;
  };
  fast_tile_fft<L, C, S, true>(sm, ld, st, tw);
}

// column pass (four-step pass A) with optional real pre-table: columns n2
// of x[n1 * L2 + n2] (length L), twiddle W_N^{S n2 k1}, stored in place-layout.
template <int L, int C, int S>
__global__ void __launch_bounds__(fast_threads<L, C>()) kc_col(const double2* __restrict__ in,
                                                              double2* __restrict__ out, int64_t N, int L2,
                                                              const double2* __restrict__ tw,
                                                              const double2* __restrict__ lo,
                                                              const double2* __restrict__ hi, int s,
                                                              const double* __restrict__ pre,
                                                              const double2* __restrict__ twQ, int Q) {
  pdl_enter();  // programmatic dependent launch: wait for the producer grid
  extern __shared__ double2 sm[];
  const int c0 = blockIdx.x * C;
  const int64_t base = (int64_t)blockIdx.y * N;
  auto ld = [&](int i, int c) -> double2 {
    const int64_t idx = (int64_t)i * L2 + c0 + c;
    double2 v = in[base + idx];
    if (pre) v = rscale(v, __ldg(&pre[idx]));
    return v;
  };
  auto st = [&](int k1, int c, double2 v) { out[base + (int64_t)k1 * L2 + c0 + c] = v; };
  const FourStepTw<S> pt{lo, hi, s, twQ, Q, c0, -1};
  fast_tile_fft<L, C, S, true>(sm, ld, st, tw, pt);
}

// ------------------------------------------------------------ host side

// rows per tile: 8, or fewer so that a 2PC-point tile stays within 4096 elements
template <int PC>
constexpr int chain_cols() { return (2 * PC * 8 <= 4096) ? 8 : 4096 / (2 * PC); }

template <typename K>
static int chain_attr(K kernel, size_t bytes) {
  if (bytes > 48 * 1024) NFFT_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  return NFFT45_OK;
}

struct ChainTabs {
  const double2 *twR, *twC, *tw2C;  // tile twiddles for lengths PR, PC and 2PC
  const FftTables *tP, *tN;         // four-step twiddles for P and n = 2P
};

// W_Q table (Q = N / last-pass stride) for the four-step post twiddles
static const double2* q_table(int64_t Q, cudaStream_t st, int* status) {
  const FftTables* t = fft_tables(Q, st, status);
  return t ? t->tw : nullptr;
}

static int chain_tables(int64_t PR, int64_t PC, ChainTabs* t, cudaStream_t st) {
  int status = NFFT45_OK;
  const FftTables* a = fft_tables(PR, st, &status);
  if (!a) return status;
  const FftTables* b = fft_tables(PC, st, &status);
  if (!b) return status;
  const FftTables* c = fft_tables(2 * PC, st, &status);
  if (!c) return status;
  t->twR = a->tw;
  t->twC = b->tw;
  t->tw2C = c->tw;
  t->tP = fft_tables(PR * PC, st, &status);
  if (!t->tP) return status;
  t->tN = fft_tables(2 * PR * PC, st, &status);
  if (!t->tN) return status;
  return NFFT45_OK;
}

template <int PR, int PC>
struct Chain {
  static constexpr int C = chain_cols<PC>();
  static constexpr int64_t P = (int64_t)PR * PC;

  // colFFT over a [len = rows*L2] signal: rows of length L2, columns of length L
  template <int L, int S>
  static int col(const double2* in, double2* out, int64_t batch, int64_t N, int L2, const double2* tw,
                 const FftTables* t4, const double* pre, cudaStream_t st) {
    // columns per tile: a power of two (it must divide L2) keeping L * CC <= 4096
    constexpr int CC = (L * 8 <= 4096) ? 8 : (L * 4 <= 4096 ? 4 : (L * 2 <= 4096 ? 2 : 1));
    auto chain_col = kc_col<L, CC, S>;
    constexpr size_t smem = fast_smem<L, CC>();
    NFFT_CHECK(chain_attr(chain_col, smem));
    constexpr int T = fast_threads<L, CC>();
    const int64_t Q = N / last_stride<L>();
    int status = NFFT45_OK;
    const double2* twQ = q_table(Q, st, &status);
    if (!twQ) return status;
    dim3 grid((unsigned)(L2 / CC), (unsigned)batch);
    LAUNCH_PDL(chain_col, grid, T, smem, st, in, out, N, L2, tw, t4->lo, t4->hi, t4->s, pre, twQ, (int)Q);
    return NFFT45_OK;
  }

  static int band(const double2* T_, double2* U, int64_t batch, const ChainTabs& t, const double* deconv,
                  const double* decay, const double* dd, const double2* sub, cudaStream_t st,
                  double2* rsave = nullptr) {
    auto chain_band = kc_band<PR, PC, C>;
    constexpr size_t smem = fast_smem<2 * PC, C>();
    NFFT_CHECK(chain_attr(chain_band, smem));
    constexpr int T = fast_threads<2 * PC, C>();
    const int64_t Q = P / last_stride<PC, HalfTr<PC>>();
    int status = NFFT45_OK;
    const double2* twQ = q_table(Q, st, &status);
    if (!twQ) return status;
    dim3 grid((unsigned)(PR / C), (unsigned)batch);
    LAUNCH_PDL(chain_band, grid, T, smem, st, T_, U, t.tw2C, t.twC, t.tP->lo, t.tP->hi, t.tP->s, deconv, decay, dd, sub,
           twQ, (int)Q, rsave);
    return NFFT45_OK;
  }

  static int mid(const double2* U, double2* Z, int64_t batch, const ChainTabs& t, const double2* ks,
                 cudaStream_t st) {
    auto chain_mid = kc_mid<PR, PC, C>;
    constexpr size_t smem = fast_smem<PR, C>();
    NFFT_CHECK(chain_attr(chain_mid, smem));
    constexpr int T = fast_threads<PR, C>();
    const int64_t Q = P / last_stride<PR>();
    int status = NFFT45_OK;
    const double2* twQ = q_table(Q, st, &status);
    if (!twQ) return status;
    dim3 grid((unsigned)(PC / C), (unsigned)batch);
    LAUNCH_PDL(chain_mid, grid, T, smem, st, U, Z, t.twR, t.tP->lo, t.tP->hi, t.tP->s, ks, twQ, (int)Q);
    return NFFT45_OK;
  }

  static int pad(const double2* Z, double2* Y, int64_t batch, const ChainTabs& t, const double* coef,
                 const double* deconv, const double* cd, const double2* xsub, double2* xout, cudaStream_t st) {
    auto chain_pad = kc_pad<PR, PC, C>;
    constexpr size_t smem = fast_smem<2 * PC, C>();
    NFFT_CHECK(chain_attr(chain_pad, smem));
    constexpr int T = fast_threads<2 * PC, C>();
    const int64_t Q = 2 * P / last_stride<2 * PC>();
    int status = NFFT45_OK;
    const double2* twQ = q_table(Q, st, &status);
    if (!twQ) return status;
    dim3 grid((unsigned)(PR / C), (unsigned)batch);
    LAUNCH_PDL(chain_pad, grid, T, smem, st, Z, Y, t.twC, t.tw2C, t.tN->lo, t.tN->hi, t.tN->s, coef, deconv, cd, xsub,
           xout, twQ, (int)Q);
    return NFFT45_OK;
  }

  // rows of length L (rows of them), output index row + R1 k
  template <int L, int S>
  static int row(const double2* in, double2* out, int64_t batch, int64_t len, int64_t R1, int rows,
                 const double2* tw, const double* post, const double2* xsub, cudaStream_t st) {
    auto chain_row = kc_row<L, C, S>;
    constexpr size_t smem = fast_smem<L, C>();
    NFFT_CHECK(chain_attr(chain_row, smem));
    constexpr int T = fast_threads<L, C>();
    dim3 grid((unsigned)(rows / C), (unsigned)batch);
    LAUNCH_PDL(chain_row, grid, T, smem, st, in, out, len, R1, tw, post, xsub);
    return NFFT45_OK;
  }
};

// Buffers for one chained solve (all [batch][len], stream-ordered scratch).
struct ChainBufs {
  double2 *H, *U, *Z;
};

template <int PR, int PC>
static int t5_front(const ChainPlanView& pv, const double2* s_or_r, int64_t batch, NodeFactor f, const double2* sub,
                    const ChainTabs& t, ChainBufs& b, cudaStream_t st) {
  using Ch = Chain<PR, PC>;
  constexpr int64_t P = Ch::P, n = 2 * P;
  Window win = Window::make(kFastM);
  NFFT_CHECK(spread(*pv.g, n, win, s_or_r, batch, f, b.H, st));
  NFFT_CHECK((Ch::template col<PR, -1>(b.H, b.H, batch, n, 2 * PC, t.twR, t.tN, nullptr, st)));
  NFFT_CHECK(Ch::band(b.H, b.U, batch, t, pv.deconv, pv.decay, pv.dd, sub, st));
  NFFT_CHECK(Ch::mid(b.U, b.Z, batch, t, pv.ks, st));
  return NFFT45_OK;
}

template <int PR, int PC>
static int chain_solve(const ChainPlanView& pv, int kind, const double2* data, int64_t batch, int passes,
                       double2* out, double* norms, cudaStream_t st) {
  using Ch = Chain<PR, PC>;
  constexpr int64_t P = Ch::P, n = 2 * P;
  ChainTabs t;
  NFFT_CHECK(chain_tables(PR, PC, &t, st));
  Window win = Window::make(kFastM);
  const GridDev& g = *pv.g;
  double2* base = nullptr;
  const size_t need = sizeof(double2) * batch * (n + P + P + n + P);
  NFFT_CUDA(cudaMallocAsync(&base, need, st));
  ChainBufs b;
  b.H = base;
  b.U = b.H + batch * n;
  b.Z = b.U + batch * P;
  double2* Y = b.Z + batch * P;    // [batch][n]
  double2* R = Y + batch * n;      // [batch][P] residual
  int status = NFFT45_OK;
  auto run = [&]() -> int {
    if (kind == 5) {
      NodeFactor fc5{pv.c5, 0.0, 0};
      NFFT_CHECK((t5_front<PR, PC>(pv, data, batch, fc5, nullptr, t, b, st)));
      for (int pass = 0; pass <= passes; pass++) {
        const bool last = (pass == passes);
        const double2* xsub = pass > 0 ? out : nullptr;
        if (last) {
          // K5: S = rowFFT_P(Z) * coef  (or x - S)
          NFFT_CHECK((Ch::template row<PC, -1>(b.Z, out, batch, P, PR, PR, t.twC, pv.coef, xsub, st)));
        } else {
          // K5+: x (= S*coef or x - S*coef) stored, padded into IFFT_2P (type-2 of x)
          NFFT_CHECK(Ch::pad(b.Z, Y, batch, t, pv.coef, pv.deconv, pv.cd, xsub, out, st));
          NFFT_CHECK((Ch::template row<PR, +1>(Y, b.H, batch, n, 2 * PC, 2 * PC, t.twR, nullptr, nullptr, st)));
          NodeFactor ph{nullptr, (double)(P / 2), +1};
          NFFT_CHECK(gather(g, n, win, b.H, batch, ph, data, R, st));  // r = type2(x) - s
          if (norms) NFFT_CHECK(row_norms(R, P, batch, norms + (int64_t)pass * batch, st));
          NFFT_CHECK((t5_front<PR, PC>(pv, R, batch, fc5, nullptr, t, b, st)));
        }
      }
    } else {
      // type 4: K1' colIFFT_P * decay -> K2' -> K3' -> K4' -> gather * c4
      auto back = [&](const double2* A_or_r, double2* dst, const double2* xsub, bool from_cols) -> int {
        if (from_cols)
          NFFT_CHECK((Ch::template col<PC, +1>(A_or_r, b.U, batch, P, PR, t.twC, t.tP, pv.decay, st)));
        NFFT_CHECK(Ch::mid(b.U, b.Z, batch, t, pv.ks, st));
        NFFT_CHECK(Ch::pad(b.Z, Y, batch, t, pv.coef, pv.deconv, pv.cd, nullptr, nullptr, st));
        NFFT_CHECK((Ch::template row<PR, +1>(Y, b.H, batch, n, 2 * PC, 2 * PC, t.twR, nullptr, nullptr, st)));
        NodeFactor fc4{pv.c4, 0.0, 0};
        return gather_mode(g, n, win, b.H, batch, fc4, xsub, xsub ? 2 : 0, dst, st);
      };
      NFFT_CHECK(back(data, out, nullptr, true));
      for (int pass = 0; pass < passes; pass++) {
        // r = type1(x) - A, then r*decay -> IFFT_P column pass (fused in K3)
        NodeFactor ph{nullptr, (double)(P / 2), -1};
        NFFT_CHECK(spread(g, n, win, out, batch, ph, b.H, st));
        NFFT_CHECK((Ch::template col<PR, -1>(b.H, b.H, batch, n, 2 * PC, t.twR, t.tN, nullptr, st)));
        // passes >= 2: the band epilogue also stores r itself, whose norms feed the
        // NonConvergence check (inverse.py:154-159)
        NFFT_CHECK(Ch::band(b.H, b.U, batch, t, pv.deconv, pv.decay, pv.dd, data, st, norms ? R : nullptr));
        if (norms) NFFT_CHECK(row_norms(R, P, batch, norms + (int64_t)pass * batch, st));
        NFFT_CHECK(back(nullptr, out, out, false));
      }
    }
    return NFFT45_OK;
  };
  status = run();
  cudaFreeAsync(base, st);
  return status;
}

bool chain_supported(int64_t P, int m) {
  if (m != kFastM) return false;
  switch (P) {
    case 1024: case 4096: case 16384: case 65536: case 262144: case 1048576:  // PR = PC
    case 2048: case 8192: case 32768: case 131072: case 524288:               // PR = 2 PC
    case 3072: case 12288: case 49152: case 196608: case 786432:              // PR = 3 * 2^a
      return true;
  }
  return false;
}

static bool batch_minor(int64_t batch) {
  static const bool no_bm = getenv("NFFT45_NO_BATCH_MINOR") != nullptr;  // A/B switch
  return batch >= 16 && !no_bm;
}

bool chain_usable(int64_t P, int m, int64_t batch) {
  if (m != kFastM) return false;
  return chain_supported(P, m) || (batch_minor(batch) && chain_bm_supported(P));
}

int chain_run(const ChainPlanView& pv, int kind, const double2* data, int64_t batch, int passes, double2* out,
              double* norms, cudaStream_t st) {
  if (batch_minor(batch) && chain_bm_supported(pv.P)) return chain_run_bm(pv, kind, data, batch, passes, out, norms, st);
  switch (pv.P) {
    case 1024: return chain_solve<32, 32>(pv, kind, data, batch, passes, out, norms, st);
    case 2048: return chain_solve<64, 32>(pv, kind, data, batch, passes, out, norms, st);
    case 4096: return chain_solve<64, 64>(pv, kind, data, batch, passes, out, norms, st);
    case 8192: return chain_solve<128, 64>(pv, kind, data, batch, passes, out, norms, st);
    case 16384: return chain_solve<128, 128>(pv, kind, data, batch, passes, out, norms, st);
    case 32768: return chain_solve<256, 128>(pv, kind, data, batch, passes, out, norms, st);
    case 65536: return chain_solve<256, 256>(pv, kind, data, batch, passes, out, norms, st);
    case 131072: return chain_solve<512, 256>(pv, kind, data, batch, passes, out, norms, st);
    case 262144: return chain_solve<512, 512>(pv, kind, data, batch, passes, out, norms, st);
    case 524288: return chain_solve<1024, 512>(pv, kind, data, batch, passes, out, norms, st);
    case 1048576: return chain_solve<1024, 1024>(pv, kind, data, batch, passes, out, norms, st);
    case 3072: return chain_solve<48, 64>(pv, kind, data, batch, passes, out, norms, st);
    case 12288: return chain_solve<96, 128>(pv, kind, data, batch, passes, out, norms, st);
    case 49152: return chain_solve<192, 256>(pv, kind, data, batch, passes, out, norms, st);
    case 196608: return chain_solve<384, 512>(pv, kind, data, batch, passes, out, norms, st);
    case 786432: return chain_solve<768, 1024>(pv, kind, data, batch, passes, out, norms, st);
  }
  return NFFT45_ERR_INVALID_ARGUMENT;
}

}  // namespace nfft45
