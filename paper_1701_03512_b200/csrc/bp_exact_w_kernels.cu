// K1w: explicit leaf enumeration with per-leaf weights (any per-step
// probabilities, reference model.py:152-161 / exact.py:95).
//
// Same decomposition as K1 (bp_exact.cuh), but the inner table is ONE sorted
// list of the 2^L suffix values (no up-count classes): leaf s carries its
// suffix weight w_s = prod over the L inner steps of p_t or 1 - p_t.  The
// table is cut into groups of 8; inside a group the in-the-money leaves are a
// prefix, so the per-leaf tests (DSETP + predicated count) give n and the
// group contributes the precomputed prefix sums PA_g[n] = sum w_s v_s and
// PB_g[n] = sum w_s.  A node with prefix weight W (running product along the
// walk, middle-step weights from a table) adds W (S A + base B):
//   Asian call  S A + (Sig - N K) B          (ITM: c_s > (N K - Sig) / S)
//   Asian put  -S A - (Sig - N K) B          (ITM: c_s < same)
//   float lb    S A + Mx (1 - B) - S E       (ITM: mx_s > Mx / S), E = sum_s w_s e_s
//   fixed lb put  K B - S A + (1 - B) max(K - Mn, 0)   (ITM: mn_s < min(Mn, K) / S)
//   euro call   S A - K B                    (ITM: e_s > K / S)
//   euro put    K B - S A                    (ITM: e_s < K / S)
// (the inner weights sum to 1: B of "all leaves" is 1).
#include "bp_kernels.h"
#include "bp_exact_w.cuh"

namespace bp {

template <bool GT>
__device__ __forceinline__ void wleaf_test(int& n, double x, double th) {
  if (GT)
    asm("{.reg .pred p; setp.gt.f64 p, %1, %2; @p add.s32 %0, %0, 1;}" : "+r"(n) : "d"(x), "d"(th));
  else
    asm("{.reg .pred p; setp.lt.f64 p, %1, %2; @p add.s32 %0, %0, 1;}" : "+r"(n) : "d"(x), "d"(th));
}

// one table slot, NP nodes: every leaf tested once per node
template <int L, int NP, int SLOT, bool GT>
__device__ __forceinline__ void wleaf_block(const double2* __restrict__ tb, const double2* __restrict__ gp,
                                            const double (&th)[NP], double (&A)[NP], double (&B)[NP]) {
  constexpr int NG = (1 << L) / kWGroup, NCH = kWGroup / kWChain;
#pragma unroll
  for (int g = 0; g < NG; ++g) {
    int nc[NP][NCH];  // independent count chains; their sum is the group's ITM prefix length
#pragma unroll
    for (int p = 0; p < NP; ++p)
#pragma unroll
      for (int c = 0; c < NCH; ++c) nc[p][c] = 0;
#pragma unroll
    for (int j = 0; j < kWGroup; ++j) {
      const int i = SLOT * (1 << L) + kWGroup * g + j;
      const double2 v = tb[i >> 1];
      const double x = (i & 1) ? v.y : v.x;
#pragma unroll
      for (int p = 0; p < NP; ++p) wleaf_test<GT>(nc[p][j / kWChain], x, th[p]);
    }
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      int n = 0;
#pragma unroll
      for (int c = 0; c < NCH; ++c) n += nc[p][c];
      const double2 q = gp[g * (kWGroup + 1) + n];  // (sum w v, sum w) of the group's first n entries
      A[p] += q.x;
      B[p] += q.y;
    }
  }
}

// leaf block + node finalisation of one kind K (table slot SL) for NP nodes
template <int L, int NP, int K, int SL>
__device__ __forceinline__ void run_kind(const double2* __restrict__ tb, const double2* __restrict__ gp,
                                         const double (&th)[NP], const double (&Sn)[NP], const double (&base)[NP],
                                         const double (&Mxn)[NP], const double (&Mnn)[NP], const double (&Wn)[NP],
                                         const ExactWScalars& sc, double (&ts)[kNumKinds], double (&tc)[kNumKinds]) {
  constexpr bool GT = (K == kAC || K == kFL || K == kEC);
  double A[NP], B[NP];
#pragma unroll
  for (int p = 0; p < NP; ++p) A[p] = B[p] = 0.0;
  wleaf_block<L, NP, SL, GT>(tb, gp, th, A, B);
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    double v;
    if constexpr (K == kAC) v = fma(Sn[p], A[p], base[p] * B[p]);
    else if constexpr (K == kAP) v = -fma(Sn[p], A[p], base[p] * B[p]);
    else if constexpr (K == kFL) v = fma(Sn[p], A[p] - sc.E, Mxn[p] * (sc.Omega - B[p]));
    else if constexpr (K == kFLP) v = fma(sc.Omega - B[p], fmax(sc.K - Mnn[p], 0.0), fma(sc.K, B[p], -Sn[p] * A[p]));
    else if constexpr (K == kEC) v = fma(Sn[p], A[p], -sc.K * B[p]);
    else v = fma(sc.K, B[p], -Sn[p] * A[p]);
    comp_add(ts[K], tc[K], Wn[p] * v);
  }
}

template <int L, unsigned KM>
__global__ void __launch_bounds__(256, 3)
k_exact_w(const __grid_constant__ ExactWArgs<L> a, double2* __restrict__ unit_out) {
  constexpr int NG = (1 << L) / 8;
  constexpr bool kAC_ = (KM >> kAC) & 1, kAP_ = (KM >> kAP) & 1, kFL_ = (KM >> kFL) & 1,
                 kFLP_ = (KM >> kFLP) & 1, kEC_ = (KM >> kEC) & 1, kEP_ = (KM >> kEP) & 1;
  constexpr int NT = (int)kAC_ + (int)kAP_ + (int)kFL_ + (int)kFLP_ + (int)kEC_ + (int)kEP_;
  static_assert(NT >= 1 && NT <= 2, "one or two kinds per launch");
  // slots in kind-bit order EC, EP, AP, FLP, AC, FL
  constexpr int sEC = 0, sEP = (int)kEC_, sAP = sEP + (int)kEP_, sFLP = sAP + (int)kAP_, sAC = sFLP + (int)kFLP_,
                sFL = sAC + (int)kAC_;
  constexpr int NP = (NT == 2) ? 2 : 4;

  __shared__ double2 sgp[NT][NG * (kWGroup + 1)];
  for (int t = 0; t < NT; ++t)
    for (int i = threadIdx.x; i < NG * (kWGroup + 1); i += blockDim.x) sgp[t][i] = a.gp[t][i];
  __syncthreads();

  const ExactWScalars& sc = a.s;
  const int lane = threadIdx.x & 31;
  const unsigned long long warp_global = (blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x) >> 5;
  const unsigned long long n_warps = (gridDim.x * (unsigned long long)blockDim.x) >> 5;
  const double INF = __longlong_as_double(0x7ff0000000000000ll);

  for (unsigned long long unit = sc.unit_first + warp_global; unit < sc.unit_end; unit += n_warps) {
    double ts[kNumKinds], tc[kNumKinds];
#pragma unroll
    for (int k = 0; k < kNumKinds; ++k) { ts[k] = 0.0; tc[k] = 0.0; }
    for (unsigned long long rr = 0; rr < (1ull << sc.q); ++rr) {
      const unsigned long long tp = (((unit << sc.q) | rr) << 5) | (unsigned long long)lane;
      // prefix walk: price, running sum / max / min and the running weight
      double S = sc.S0, Sig = 0.0, Mx = 0.0, Mn = INF, W = sc.disc;
      for (int t = sc.Dp - 1; t >= 0; --t) {
        const int step = sc.Dp - 1 - t;  // 0-based step index
        const int b = (int)((tp >> t) & 1ull);
        S *= b ? sc.u : sc.d;
        Sig += S;
        Mx = fmax(Mx, S);
        Mn = fmin(Mn, S);
        W *= b ? a.p[step] : a.q[step];
      }
      for (int j0 = 0; j0 < sc.n_mid; j0 += NP) {
        double Sn[NP], Wn[NP], base[NP], Mxn[NP], Mnn[NP];
        double thC[NP], thX[NP], thN[NP], thE[NP];
#pragma unroll
        for (int p = 0; p < NP; ++p) {
          const int j = j0 + p;
          Sn[p] = S * a.mid_e[j];
          base[p] = fma(S, a.mid_c[j], Sig) - sc.NK;
          Mxn[p] = fmax(Mx, S * a.mid_mx[j]);
          Mnn[p] = fmin(Mn, S * a.mid_mn[j]);
          Wn[p] = W * a.mid_w[j];
          const double rS = 1.0 / Sn[p];
          thC[p] = -base[p] * rS;
          thX[p] = Mxn[p] * rS;
          thN[p] = fmin(Mnn[p], sc.K) * rS;
          thE[p] = sc.K * rS;
        }
        const double2* tb = reinterpret_cast<const double2*>(a.tab) + (j0 & sc.zero);  // + 0, opaque
        if (kEC_) run_kind<L, NP, kEC, sEC>(tb, sgp[sEC], thE, Sn, base, Mxn, Mnn, Wn, sc, ts, tc);
        if (kEP_) run_kind<L, NP, kEP, sEP>(tb, sgp[sEP], thE, Sn, base, Mxn, Mnn, Wn, sc, ts, tc);
        if (kAP_) run_kind<L, NP, kAP, sAP>(tb, sgp[sAP], thC, Sn, base, Mxn, Mnn, Wn, sc, ts, tc);
        if (kFLP_) run_kind<L, NP, kFLP, sFLP>(tb, sgp[sFLP], thN, Sn, base, Mxn, Mnn, Wn, sc, ts, tc);
        if (kAC_) run_kind<L, NP, kAC, sAC>(tb, sgp[sAC], thC, Sn, base, Mxn, Mnn, Wn, sc, ts, tc);
        if (kFL_) run_kind<L, NP, kFL, sFL>(tb, sgp[sFL], thX, Sn, base, Mxn, Mnn, Wn, sc, ts, tc);
      }
    }
#pragma unroll
    for (int k = 0; k < kNumKinds; ++k) {
      if (!((KM >> k) & 1)) continue;
      double s = ts[k], c = tc[k];
      warp_comp_reduce(s, c);
      if (lane == 0) unit_out[unit * kNumKinds + k] = make_double2(s, c);
    }
  }
}

#define BP_W_KMS(X)                                                                                      \
  X((1u << kAC)) X((1u << kAP)) X((1u << kFL)) X((1u << kFLP)) X((1u << kEC)) X((1u << kEP))           \
  X(((1u << kAC) | (1u << kFL)))

cudaError_t launch_exact_w(unsigned km, const void* args, int grid, cudaStream_t st, double2* unit_out) {
  const ExactWArgs<8>& a = *static_cast<const ExactWArgs<8>*>(args);
#define BP_CASE(KMV) \
  if (km == (KMV)) { k_exact_w<8, (KMV)><<<grid, 256, 0, st>>>(a, unit_out); return cudaGetLastError(); }
  BP_W_KMS(BP_CASE)
#undef BP_CASE
  return cudaErrorInvalidValue;
}

int occupancy_exact_w(unsigned km) {
  int n = 0;
#define BP_CASE(KMV) \
  if (km == (KMV)) { cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_exact_w<8, (KMV)>, 256, 0); return n; }
  BP_W_KMS(BP_CASE)
#undef BP_CASE
  return 0;
}

}  // namespace bp
