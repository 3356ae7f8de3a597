// Structured element solve for RT2 / RT3 hexahedra: one 512-thread CTA per
// cell (n = 108 / 240 local dofs, nF = 54 / 96 face dofs).
//
// Same mathematics as kern_warp.cu (fp64 V = A0^-1 [E_F | f_T]; fp32 first-order
// correction C = V_F^T (Delta32 V); a-posteriori order control), organised for
// elements whose n x n matrices do not fit on chip:
//   phase V  : V in row blocks (X rows staged per block), fp32 copy V32 kept in
//              shared memory (n x NCP), fp64 face rows to a per-CTA scratch
//   phase C  : Delta32 generated in row blocks of IB rows (stored transposed),
//              Y_I = Delta_I V32 (smem), C += V32_I^T Y_I with C held in registers
//              (a 6x7 / 3x4 tile per thread) across all blocks
//   scatter  : per-cell tables, H = V_F - C, red-black like the other paths.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <type_traits>

#include "hdr_device.cuh"
#include "kernels.hpp"
#include "umma.cuh"

namespace hdr {
namespace {

template <int K>
struct Big {
  static constexpr int DIM = 3;
  static constexpr int DPF = (K + 1) * (K + 1);
  static constexpr int NF = 6 * DPF;
  static constexpr int NINT = 3 * K * DPF;
  static constexpr int N = NF + NINT;
  static constexpr int R = (K + 1) * (K + 1) * (K + 1);
  static constexpr int NC = NF + 1;
  static constexpr int NCP = (NC + 3) & ~3;
  static constexpr int IB = (K == 3) ? 48 : 54;  // rows per block: divides N and NINT (interior / face blocks)
  static constexpr int NB = N / IB;
  // fp64 tensor-core (DMMA m8n8k4) phase V: row strides chosen so that each
  // half-warp's fragment loads hit 16 distinct bank pairs (2 wavefronts per load)
  static constexpr int NZ = ((NC + 7) / 8 * 8 + 11) / 16 * 16 + 4;  // z (RP x NZ), NZ = 4 mod 16, >= 8 CT
  static constexpr int RP = (R + 3) & ~3;            // K of the V product, padded to the MMA's 4
  static constexpr int RS = (RP + 11) / 16 * 16 + 4; // xi (IBP x RS), RS = 4 mod 16
  static constexpr int IBP = (IB + 7) & ~7;          // row block padded to the MMA's 8

  // thread tiles: V / Y blocks (IB x NC), C (NF x NC)
  static constexpr int VT_M = (K == 3) ? 4 : 3, VT_N = (K == 3) ? 6 : 3;
  static constexpr int CT_M = (K == 3) ? 6 : 3, CT_N = (K == 3) ? 7 : 4;
  static constexpr int NS = 6;
  // tensor-core (tcgen05, 3xTF32) shapes of the first-order correction:
  //   Y^T (128 x NY) = V^T (128 x KP) Delta^T (KP x NY);  C^T (128 x NFP) = Y^T (128 x KP) V_F (KP x NFP)
  //   (the Delta tables keep MP = MT1 * 128 rows per chunk; rows >= N are zero)
  static constexpr int MT1 = (N + 127) / 128, MP = MT1 * 128;
  static constexpr int NP = (NC + 15) / 16 * 16, KP = (N + 15) / 16 * 16;
  static constexpr int NY = KP, NFP = (NF + 15) / 16 * 16;
  static constexpr int KC2 = 32, NCH2 = (KP + KC2 - 1) / KC2;  // C^T product chunks
  static constexpr int KC = 16;  // K per operand chunk (two K=8 MMA steps)
  static constexpr int TCOLS_USED = NY + NFP;
  static constexpr int TCOLS = TCOLS_USED <= 32 ? 32 : TCOLS_USED <= 64 ? 64 : TCOLS_USED <= 128 ? 128 : TCOLS_USED <= 256 ? 256 : 512;
};

constexpr int kThreads = 512;

#ifdef HDR_BIG_TIMING  // phase cycle counters of CTA 0 (variant builds only: make EXTRA=-DHDR_BIG_TIMING)
__device__ unsigned long long g_big_prof[32];
#define BIG_T(slot)                                                         \
  do {                                                                      \
    if (blockIdx.x == 0 && threadIdx.x == 0) {                              \
      const long long now_ = clock64();                                     \
      g_big_prof[slot] += static_cast<unsigned long long>(now_ - t_last_); \
      t_last_ = now_;                                                       \
    }                                                                       \
  } while (0)
#else
#define BIG_T(slot) \
  do {              \
  } while (0)
#endif

template <int K>
struct BigSmem {
  using B = Big<K>;
  float v32[B::N * B::NCP];
  union U {
    struct {
      double z[B::RP * B::NZ];
      double xi[2][B::IBP * B::RS];  // double-buffered row blocks of X
    } pv;
    struct {
      float dt[B::N * B::IB];  // Delta32 block transposed: dt[l * IB + ii]
      float y[B::IB * B::NCP];
    } pc;
    struct {  // tcgen05 operand chunks (canonical K-major, no swizzle), hi / lo tf32 parts
      float ahi[128 * B::KC], alo[128 * B::KC];    // V^T / Y^T chunk (M = 128)
      float bhi[B::NY * B::KC], blo[B::NY * B::KC];  // Delta chunk (N = NY) / V_F chunk (N = NFP)
    } tc[2];    // double-buffered: chunk c + 1 is generated while the MMAs of chunk c run
    struct {  // the C^T product's operand chunks, K = KC2 (fewer, longer chunks)
      float ahi[128 * B::KC2], alo[128 * B::KC2];    // Y^T chunk (from TMEM)
      float bhi[B::NFP * B::KC2], blo[B::NFP * B::KC2];  // V_F chunk
    } tc2[2];
    float csm[B::NF * B::NCP];  // the correction C (NF x NC) for the scatter
  } u;
  double f[B::N], nf[B::N], s[B::R];
  long long rstart[B::NS];
  int rlen[B::NS], grow[B::NS], rank[B::NS * B::NS];
  float red[2 * kThreads / 32];
  int order;
  int exact;  // the cell is rejected: zeros here, the exact path (kern_exact.cu) adds it
  uint64_t mbar[2];
  uint32_t tmem;
};

template <int K>
constexpr int64_t big_scratch_doubles() {
  using B = Big<K>;
  // vf (NF x NC fp64) + Y (N x NCP fp32) + T (N x NCP fp32)
  return static_cast<int64_t>(B::NF) * B::NC + static_cast<int64_t>(B::N) * B::NCP + 16;
}

// x = hi + lo with hi, lo tf32 (low 13 mantissa bits zero; hi rounded half away
// from zero like cvt.rna): integer ops only (the tensor core reads the top 19
// bits; x - hi is exact in fp32)
__device__ __forceinline__ void tf32_split(float x, float& hi, float& lo) {
  hi = __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
  const float r = x - hi;
  lo = __uint_as_float((__float_as_uint(r) + 0x1000u) & 0xFFFFE000u);
}

// One row block [i0, i0 + IB) of [V | w] = (base + X z) / beta, register tiles
// in T (double for the face rows, float for the interior rows).
__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// One row block [i0, i0 + IB) of [V | w] = (base + X z) / beta on the fp64
// tensor cores: warp tiles of 8 rows x 8 columns, K = RP in steps of 4
// (fragments: a = xi[row = lane/4][k = lane%4], b = z[k = lane%4][col = lane/4],
// d = (row lane/4, cols 2 (lane%4) + {0, 1})).  Face blocks: V_FF is symmetric,
// only tiles reaching the lower triangle are computed, the rest mirrored.
template <int K>
__device__ __forceinline__ void v_block(BigSmem<K>& sm, const Fixed& fx, int i0, double ib, double* vf) {
  using B = Big<K>;
  constexpr int N = B::N, NF = B::NF, NC = B::NC, NCP = B::NCP, NINT = B::NINT, IB = B::IB, NZ = B::NZ, RS = B::RS;
  constexpr int RT = B::IBP / 8, CT = (NC + 7) / 8;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool face = i0 >= NINT;
  const int pb = i0 - NINT;
  const double* xi = sm.u.pv.xi[(i0 / IB) & 1];
  const double* z = sm.u.pv.z;
  for (int t = warp; t < RT * CT; t += kThreads / 32) {
    const int rt = t / CT, ct = t - rt * CT;
    if (face && ct * 8 + 7 < NF && ct * 8 > pb + rt * 8 + 7) continue;  // strictly above the diagonal (no w column)
    const int r = rt * 8 + (lane >> 2), c0 = ct * 8 + 2 * (lane & 3);
    const int row = i0 + r;
    const bool rok = r < IB;
    double base[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int col = c0 + q;
      base[q] = !rok || col >= NC ? 0.0
                : (col < NF ? __ldg(fx.N0 + static_cast<int64_t>(row) * N + NINT + col) : sm.nf[row]);
    }
    const double* ap = xi + (rt * 8 + (lane >> 2)) * RS + (lane & 3);
    const double* bp = z + (lane & 3) * NZ + ct * 8 + (lane >> 2);
    // fragments loaded in batches of 8 k-steps ahead of their MMAs; two
    // accumulator pairs (even / odd k-steps) halve the dependent MMA chain
    constexpr int KS = B::RP / 4, KB = KS < 8 ? KS : 8;
    double d0 = 0.0, d1 = 0.0, e0 = 0.0, e1 = 0.0;
#pragma unroll
    for (int k0 = 0; k0 < KS; k0 += KB) {
      double av[KB], bv[KB];
#pragma unroll
      for (int u = 0; u < KB; ++u) {
        av[u] = k0 + u < KS ? ap[4 * (k0 + u)] : 0.0;
        bv[u] = k0 + u < KS ? bp[4 * (k0 + u) * NZ] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < KB; ++u) {
        if (u & 1) dmma_8x8x4(e0, e1, av[u], bv[u]);
        else dmma_8x8x4(d0, d1, av[u], bv[u]);
      }
    }
    d0 += e0;
    d1 += e1;
    if (!rok) continue;
    const double dv[2] = {d0, d1};
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int col = c0 + q;
      if (col >= NC) continue;
      if (face && col < NF && col > pb + r) continue;
      const double v = (base[q] + dv[q]) * ib;
      sm.v32[row * NCP + col] = static_cast<float>(v);
      if (face) {
        vf[(row - NINT) * NC + col] = v;
        if (col < NF && col < pb + r) {  // mirror (col, row) of the symmetric face block
          const int p = pb + r;
          sm.v32[(NINT + col) * NCP + p] = static_cast<float>(v);
          vf[col * NC + p] = v;
        }
      }
    }
  }
}

// First-order correction on the tensor cores (3xTF32), in transposed form so
// that the intermediate never has to be transposed:
//   Y^T = V^T Delta^T  (M = 128 columns c of [V | w], N = NY rows of Delta, in TMEM)
//   C^T = Y^T V_F      (M = 128, N = NFP face columns; A = Y^T chunks copied from
//                       TMEM: lane c holds row c, i.e. exactly the A layout)
// operands generated chunk by chunk (K = 16) straight into the canonical
// shared-memory layout; one thread issues the MMAs, everyone waits on the
// commit mbarrier before the buffers are refilled.  C -> sm.u.csm.
template <int K>
__device__ void correction_tc(BigSmem<K>& sm, const Fixed& fx, double a, double b, uint32_t& ph) {
  using B = Big<K>;
  constexpr int N = B::N, NF = B::NF, NC = B::NC, NCP = B::NCP;
  constexpr int MP = B::MP, KP = B::KP, KC = B::KC, NY = B::NY, NFP = B::NFP, NCH = KP / KC;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t tY = sm.tmem, tC = sm.tmem + NY;
  constexpr uint32_t idesc1 = umma::idesc_tf32(128, NY), idesc2 = umma::idesc_tf32(128, NFP);
  constexpr uint32_t lbo_a = (128 / 8) * 128, lbo_b1 = (NY / 8) * 128, lbo_b2 = (NFP / 8) * 128;
  auto wait_buf = [&](int bf) {  // the MMAs that last read buffer bf are done
    umma::mbar_wait(&sm.mbar[bf], (ph >> bf) & 1u);  // phase bits in a register (no local memory)
    ph ^= 1u << bf;
    umma::fence_after();
  };
  auto issue = [&](auto& T, int c, uint32_t tD, uint32_t idesc, uint32_t lbo_b) {
    umma::fence_after();
    for (int ks = 0; ks < KC / 8; ++ks)
      for (int term = 0; term < 3; ++term) {
        const float* aop = term == 2 ? T.alo : T.ahi;
        const float* bop = term == 1 ? T.blo : T.bhi;
        const uint64_t ad = umma::smem_desc(umma::smem_u32(aop) + ks * 2 * lbo_a, lbo_a, 128);
        const uint64_t bd = umma::smem_desc(umma::smem_u32(bop) + ks * 2 * lbo_b, lbo_b, 128);
        umma::mma_tf32(tD, ad, bd, idesc, c > 0 || ks > 0 || term > 0);
      }
  };
  // ---- Y^T = V^T Delta^T.  Delta's inputs come from the chunk-ordered tables
  // (dtab: {D, M} fp64, etab: {E, Ma} fp32; zero padded), coalesced, and the
  // next chunk's loads are issued as soon as the current chunk is generated.
  constexpr int PER = MP * KC / kThreads;
  static_assert(PER * kThreads == MP * KC, "chunk entries per thread");
  const float af = static_cast<float>(a), bf32 = static_cast<float>(b);
  double2 dm[PER];
  float2 em[PER];
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    dm[i] = __ldg(fx.dtab + tid + i * kThreads);
    em[i] = __ldg(fx.etab + tid + i * kThreads);
  }
  for (int c = 0; c < NCH; ++c) {
    const int bf = c & 1, kc = c * KC;
    auto& T = sm.u.tc[bf];
#ifdef HDR_BIG_TIMING
    long long tq = clock64();
#define BIG_Q(slot)                                                      \
  if (blockIdx.x == 0 && threadIdx.x == 0) {                             \
    const long long nq_ = clock64();                                     \
    g_big_prof[slot] += static_cast<unsigned long long>(nq_ - tq);       \
    tq = nq_;                                                            \
  }
#else
#define BIG_Q(slot)
#endif
    if (c >= 2) wait_buf(bf);
    BIG_Q(8);
    const int64_t q0 = static_cast<int64_t>(c + 1) * MP * KC + tid;
#pragma unroll
    for (int i = 0; i < PER; ++i) {  // lane -> (n % 8, k % 4): the 32 lanes store to 32 banks
      const int g = warp + 16 * i, m = 8 * (g >> 2) + (lane >> 2), k = 4 * (g & 3) + (lane & 3);
      if (8 * (g >> 2) < NY) {  // else padding rows of the table (warp-uniform)
        // delta (exact rounding error of the combine) in fp64; alpha E + beta Ma in fp32
        double p1, e1, p2, e2, sm_, e3;
        two_prod(a, dm[i].x, p1, e1);
        two_prod(b, dm[i].y, p2, e2);
        two_sum_fast(p1, p2, sm_, e3);
        const float x = fmaf(af, em[i].x, fmaf(bf32, em[i].y, static_cast<float>(-((e1 + e2) + e3))));
        const uint32_t off = umma::kmajor_offset(m, k, NY) >> 2;
        tf32_split(x, T.bhi[off], T.blo[off]);
      }
      if (c + 1 < NCH) {  // entry i of the next chunk in flight as soon as its registers are free
        dm[i] = __ldg(fx.dtab + q0 + i * kThreads);
        em[i] = __ldg(fx.etab + q0 + i * kThreads);
      }
    }
    BIG_Q(9);
    for (int g = warp; g < 64; g += 16) {  // V^T chunk: lane -> (c % 8, k % 4)
      const int m = 8 * (g >> 2) + (lane >> 2), k = 4 * (g & 3) + (lane & 3), row = kc + k;
      const float x = (m < NC && row < N) ? sm.v32[row * NCP + m] : 0.f;
      const uint32_t off = umma::kmajor_offset(m, k, 128) >> 2;
      tf32_split(x, T.ahi[off], T.alo[off]);
    }
    BIG_Q(10);
    umma::fence_proxy_async();
    __syncthreads();
    BIG_Q(11);
    if (tid == 0) {
      issue(T, c, tY, idesc1, lbo_b1);
      umma::commit(&sm.mbar[bf]);
    }
  }
  wait_buf(NCH & 1);        // chunk NCH - 2
  wait_buf((NCH - 1) & 1);  // chunk NCH - 1: Y^T complete
#ifdef HDR_BIG_TIMING
  if (blockIdx.x == 0 && threadIdx.x == 0) g_big_prof[13] = clock64();
#endif
  // ---- C^T = Y^T V_F  (A operand: Y^T chunk from TMEM; lane c holds row c), K = 32 per chunk
  constexpr int KC2 = B::KC2, NCH2 = B::NCH2;
  for (int c = 0; c < NCH2; ++c) {
    const int bf = c & 1, kc = c * KC2;
    auto& T = sm.u.tc2[bf];
    if (c >= 2) wait_buf(bf);
    {  // the 4 warps of lane quadrant q = warp % 4 take 8 columns each (columns >= N: zero)
      const int q = warp & 3, k0 = 8 * (warp >> 2), m = 32 * q + lane;
      float v[8];
      if (kc + k0 < N) {
        umma::tmem_ld8(tY + (static_cast<uint32_t>(32 * q) << 16) + kc + k0, v);
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = 0.f;
      }
      float hi[8], lo[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) tf32_split(kc + k0 + j < N ? v[j] : 0.f, hi[j], lo[j]);
      const uint32_t off0 = umma::kmajor_offset(m, k0, 128) >> 2, off1 = umma::kmajor_offset(m, k0 + 4, 128) >> 2;
      *reinterpret_cast<float4*>(T.ahi + off0) = make_float4(hi[0], hi[1], hi[2], hi[3]);
      *reinterpret_cast<float4*>(T.alo + off0) = make_float4(lo[0], lo[1], lo[2], lo[3]);
      *reinterpret_cast<float4*>(T.ahi + off1) = make_float4(hi[4], hi[5], hi[6], hi[7]);
      *reinterpret_cast<float4*>(T.alo + off1) = make_float4(lo[4], lo[5], lo[6], lo[7]);
    }
    for (int g = warp; g < NFP / 8 * (KC2 / 4); g += 16) {  // V_F chunk: lane -> (f % 8, k % 4)
      const int f = 8 * (g / (KC2 / 4)) + (lane >> 2), k = 4 * (g % (KC2 / 4)) + (lane & 3), row = kc + k;
      const float x = (f < NF && row < N) ? sm.v32[row * NCP + f] : 0.f;
      const uint32_t off = umma::kmajor_offset(f, k, NFP) >> 2;
      tf32_split(x, T.bhi[off], T.blo[off]);
    }
    umma::fence_proxy_async();
    umma::fence_before();
    __syncthreads();
    if (tid == 0) {
      umma::fence_after();
      for (int ks = 0; ks < KC2 / 8; ++ks)
        for (int term = 0; term < 3; ++term) {
          const float* aop = term == 2 ? T.alo : T.ahi;
          const float* bop = term == 1 ? T.blo : T.bhi;
          const uint64_t ad = umma::smem_desc(umma::smem_u32(aop) + ks * 2 * lbo_a, lbo_a, 128);
          const uint64_t bd = umma::smem_desc(umma::smem_u32(bop) + ks * 2 * lbo_b2, lbo_b2, 128);
          umma::mma_tf32(tC, ad, bd, idesc2, c > 0 || ks > 0 || term > 0);
        }
      umma::commit(&sm.mbar[bf]);
    }
  }
  wait_buf(NCH2 & 1);
  wait_buf((NCH2 - 1) & 1);
  // ---- C^T -> C in shared memory: lane c holds C^T[c][f] = C[f][c]
  {
    const int q = warp & 3, m = 32 * q + lane;
    for (int cc = 8 * (warp >> 2); cc < NFP; cc += 8 * (kThreads / 128)) {
      float v[8];
      umma::tmem_ld8(tC + (static_cast<uint32_t>(32 * q) << 16) + cc, v);
      if (m < NC)
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (cc + j < NF) sm.u.csm[(cc + j) * NCP + m] = v[j];
    }
  }
  umma::fence_before();
  __syncthreads();
}

template <int K>
__global__ void __launch_bounds__(kThreads, 1) k_hyb_big(HybArgs A, int parity, double* gws, int use_tc,
                                                         const double* pre) {
  using B = Big<K>;
  constexpr int N = B::N, NF = B::NF, NC = B::NC, NCP = B::NCP, R = B::R, NINT = B::NINT, DPF = B::DPF;
  constexpr int IB = B::IB, NS = B::NS;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  BigSmem<K>& sm = *reinterpret_cast<BigSmem<K>*>(smem_raw);
  const int tid = threadIdx.x;
  uint32_t phase = 0u;  // bit b: parity of mbar[b]
  if (use_tc) {
    if (tid == 0) {
      umma::mbar_init(&sm.mbar[0], 1);
      umma::mbar_init(&sm.mbar[1], 1);
    }
    if ((tid >> 5) == 0) umma::tmem_alloc(&sm.tmem, B::TCOLS);
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
  }
  const Fixed& fx = A.fx;
  double* vf = gws + static_cast<int64_t>(blockIdx.x) * big_scratch_doubles<K>();  // NF x NC
  float* yg = reinterpret_cast<float*>(vf + NF * NC);                               // N x NCP (Y, higher orders)
  const uint32_t cnt = static_cast<uint32_t>(parity_count(A.m));

#ifdef HDR_BIG_TIMING
  long long t_last_ = clock64();
#endif
  for (uint32_t t = blockIdx.x; t < cnt; t += gridDim.x) {
    int cc[3];
    const int e = parity_cell32(A.m, parity, t, cc);
    if (e < 0) continue;
    BIG_T(0);
    const double a = A.alpha[e], b = A.beta[e];
    const double ib = 1.0 / b;
    const double* fe = A.f + static_cast<int64_t>(e) * N;
    // scatter tables (cell geometry only) and an L2 prefetch of the shared
    // diagonal blocks' partial sums (colour 1 adds to colour 0's): made by warp 15
    // during the first V block, where it has one tile fewer than warps 0..13
    auto scatter_tables = [&](int lane_) {
    {
      unsigned lo = 0, hi = 0;
#pragma unroll
      for (int x = 0; x < 3; ++x) {
        const int cx = x == 0 ? cc[0] : (x == 1 ? cc[1] : cc[2]);
        const int Nx = static_cast<int>(x == 0 ? A.m.N[0] : (x == 1 ? A.m.N[1] : A.m.N[2]));
        lo |= static_cast<unsigned>(cx > 0) << x;
        hi |= static_cast<unsigned>(cx + 1 < Nx) << x;
      }
      for (int idx = lane_; idx < NS * NS; idx += 32) {
        const int ps = idx / NS, qs = idx - ps * NS;
        const int a_ = ps >> 1;
        const bool pin = (((ps & 1) ? hi : lo) >> a_) & 1u;
        const bool qin = (((qs & 1) ? hi : lo) >> (qs >> 1)) & 1u;
        const int ca = a_ == 0 ? cc[0] : (a_ == 1 ? cc[1] : cc[2]);
        const int na = static_cast<int>(a_ == 0 ? A.m.N[0] : (a_ == 1 ? A.m.N[1] : A.m.N[2]));
        sm.rank[idx] = (pin && qin) ? col_rank_fast(3, ps, qs, lo, hi, ca, na, false) : -1;
        if (qs == 0) {
          const int side = ps & 1;
          if (pin) {
            const int face = face_id32(A.m, a_, cc[0] + (a_ == 0 ? side : 0), cc[1] + (a_ == 1 ? side : 0),
                                       cc[2] + (a_ == 2 ? side : 0));
            const int row = A.mbase[face];
            const int64_t r0s = A.rowoff[row];
            sm.rstart[ps] = r0s;
            sm.rlen[ps] = static_cast<int>(A.rowoff[row + 1] - r0s);
            sm.grow[ps] = row;
          } else {
            sm.rstart[ps] = -1;
          }
        }
      }
    }
    __syncwarp();
    if (parity == 1)
      for (int q = lane_; q < NS * DPF * (DPF * 8 / 128 + 1); q += 32) {
        const int ps = q / (DPF * (DPF * 8 / 128 + 1)), rem = q - ps * (DPF * (DPF * 8 / 128 + 1));
        const int sub = rem / (DPF * 8 / 128 + 1), part = rem - sub * (DPF * 8 / 128 + 1);
        const int64_t rs = sm.rstart[ps];
        const int rk = sm.rank[ps * NS + ps];
        if (rs < 0 || rk < 0) continue;
        const double* line = A.hval + rs + static_cast<int64_t>(sub) * sm.rlen[ps] + rk * DPF + part * 16;
        asm volatile("prefetch.global.L2 [%0];" ::"l"(line));
      }
    };
    // ---------------------------------------------------------------- phase V (fp64)
    // X_F (rows of the face dofs) for z = s X_F^T: all loads in flight before the barrier
    constexpr int ZPT = (R * NF + kThreads - 1) / kThreads;
    double xz[ZPT];
#pragma unroll
    for (int u = 0; u < ZPT; ++u) {  // j fastest: coalesced rows of X
      const int idx = tid + u * kThreads, c = idx / R, j = idx - c * R;
      xz[u] = idx < R * NF ? __ldg(fx.X + (NINT + c) * R + j) : 0.0;
    }
    for (int i = tid; i < N; i += kThreads) sm.f[i] = fe[i];
    for (int j = tid; j < R; j += kThreads) sm.s[j] = b / fma(a, __ldg(fx.lam + j), b);
    const double* pe = pre + static_cast<int64_t>(e) * (N + R);  // [N0 f_e ; X^T f_e], batched GEMM
    for (int i = tid; i < N; i += kThreads) sm.nf[i] = pe[i];
    __syncthreads();
#pragma unroll
    for (int u = 0; u < ZPT; ++u) {
      const int idx = tid + u * kThreads, c = idx / R, j = idx - c * R;
      if (idx < R * NF) sm.u.pv.z[j * B::NZ + c] = sm.s[j] * xz[u];
    }
    for (int j = tid; j < B::RP; j += kThreads) {
      sm.u.pv.z[j * B::NZ + NF] = j < R ? sm.s[j] * pe[N + j] : 0.0;
      for (int c = (j < R ? NC : 0); c < B::NZ; ++c) sm.u.pv.z[j * B::NZ + c] = 0.0;
    }
    BIG_T(1);
    // row blocks on the fp64 tensor cores (the interior rows only feed the
    // fp32 correction and are rounded to fp32; the face rows give H0 = V_F, g0)
    {
      constexpr int XE = B::IBP * B::RS, XPT = (XE + kThreads - 1) / kThreads;
      auto xload = [&](int i0, double (&reg)[XPT]) {
#pragma unroll
        for (int u = 0; u < XPT; ++u) {
          const int idx = tid + u * kThreads, r = idx / B::RS, j = idx - r * B::RS;
          reg[u] = (idx < XE && r < IB && j < R && i0 + r < N) ? __ldg(fx.X + (i0 + r) * R + j) : 0.0;
        }
      };
      auto xstore = [&](int buf, const double (&reg)[XPT]) {
#pragma unroll
        for (int u = 0; u < XPT; ++u)
          if (tid + u * kThreads < XE) sm.u.pv.xi[buf][tid + u * kThreads] = reg[u];
      };
      double xr[XPT];
      xload(0, xr);
      xstore(0, xr);
      __syncthreads();
      for (int i0 = 0; i0 < N; i0 += IB) {
        const bool more = i0 + IB < N;
        if (more) xload(i0 + IB, xr);  // next block's X rows in flight during this block
        v_block<K>(sm, fx, i0, ib, vf);
        if (i0 == 0 && (tid >> 5) == kThreads / 32 - 1) scatter_tables(tid & 31);
        if (more) xstore(((i0 / IB) + 1) & 1, xr);
        __syncthreads();
      }
    }
    // ---------------------------------------------------------------- phase C
    // first order on the tensor cores; the CUDA-core path below is kept for
    // the (rare) cells whose a-posteriori estimate asks for a second order
    BIG_T(2);
    bool tc_done = false;
    if (use_tc) {
      correction_tc<K>(sm, fx, a, b, phase);
#ifdef HDR_BIG_TIMING
      if (blockIdx.x == 0 && threadIdx.x == 0) { g_big_prof[3] += g_big_prof[13] - t_last_; t_last_ = g_big_prof[13]; }
#endif
      BIG_T(4);
      float cmax = 0.f, hmax = 0.f;
      for (int idx = tid; idx < NF * NF; idx += kThreads) {
        const int p = idx / NF, q = idx - p * NF;
        cmax = fmaxf(cmax, fabsf(sm.u.csm[p * NCP + q]));
        hmax = fmaxf(hmax, fabsf(sm.v32[(NINT + p) * NCP + q]));
      }
      for (int o = 16; o > 0; o >>= 1) {
        cmax = fmaxf(cmax, __shfl_xor_sync(0xffffffffu, cmax, o));
        hmax = fmaxf(hmax, __shfl_xor_sync(0xffffffffu, hmax, o));
      }
      if ((tid & 31) == 0) {
        sm.red[tid >> 5] = cmax;
        sm.red[kThreads / 32 + (tid >> 5)] = hmax;
      }
      __syncthreads();
      if (tid == 0) {
        float cm = 0.f, hm = 0.f;
        for (int w = 0; w < kThreads / 32; ++w) {
          cm = fmaxf(cm, sm.red[w]);
          hm = fmaxf(hm, sm.red[kThreads / 32 + w]);
        }
        const double ratio = hm > 0.f ? static_cast<double>(cm) / hm : 0.0;
        // the tensor core's fp32 accumulation is less accurate than fp32 FMA
        // chains (eps_tc ~ 1e-6 of |C|): its C is accepted only where the
        // estimate allows it at order 1 (hdr_device.cuh struct_order); cells the
        // CUDA-core form cannot accept either go straight to the exact path
        bool ex_tc = false, ex32 = false;
        const int p = struct_order(ratio, A.p_max, A.eps_tc, ex_tc);
        struct_order(ratio, A.p_max, A.eps32, ex32);
        sm.exact = (ex32 || A.force_exact) ? 1 : 0;
        sm.order = (!ex_tc && p == 1) ? 1 : 0;
        if (A.qlog) A.qlog[e] = static_cast<float>(ratio);
        if (sm.exact) exact_push(A.xlist, A.xcount, e);
      }
      __syncthreads();
      tc_done = sm.order == 1 || sm.exact;
    } else if (tid == 0) {
      sm.exact = 0;
    }
    BIG_T(5);
    if (!tc_done) {
      constexpr int CM = B::CT_M, CN = B::CT_N;
      constexpr int CMS = (NF + CM - 1) / CM, CNS = (NC + CN - 1) / CN;
      const bool cown = tid < CMS * CNS;
      const int cm0 = cown ? (tid / CNS) * CM : 0, cn0 = cown ? (tid % CNS) * CN : 0;
      float cacc[CM][CN];
  #pragma unroll
      for (int i = 0; i < CM; ++i)
  #pragma unroll
        for (int j = 0; j < CN; ++j) cacc[i][j] = 0.f;
      int P = 1;
      for (int pass = 1; pass <= P; ++pass) {
        // right operand of this order: V32 (pass 1) or T = A0^-1 Y_prev (global, rare)
        const float* rhs = (pass == 1) ? sm.v32 : yg + N * NCP;  // T staged behind Y in scratch
        for (int i0 = 0; i0 < N; i0 += IB) {
          for (int idx = tid; idx < IB * N; idx += kThreads) {
            const int ii = idx / N, l = idx - ii * N;
            const int64_t o = static_cast<int64_t>(i0 + ii) * N + l;
            sm.u.pc.dt[l * IB + ii] = static_cast<float>(
                delta_entry(a, b, __ldg(fx.D + o), __ldg(fx.M + o), __ldg(fx.E + o), __ldg(fx.Ma + o)));
          }
          __syncthreads();
          {  // Y_I = Delta_I rhs
            constexpr int TM = B::VT_M, TN = B::VT_N;
            constexpr int TMS = (IB + TM - 1) / TM, TNS = (NC + TN - 1) / TN;
            for (int tile = tid; tile < TMS * TNS; tile += kThreads) {
              const int m0 = (tile / TNS) * TM, n0 = (tile % TNS) * TN;
              float acc[TM][TN];
  #pragma unroll
              for (int i = 0; i < TM; ++i)
  #pragma unroll
                for (int jj = 0; jj < TN; ++jj) acc[i][jj] = 0.f;
  #pragma unroll 4
              for (int l = 0; l < N; ++l) {
                float dv[TM], rv[TN];
  #pragma unroll
                for (int i = 0; i < TM; ++i) dv[i] = (m0 + i < IB) ? sm.u.pc.dt[l * IB + m0 + i] : 0.f;
  #pragma unroll
                for (int jj = 0; jj < TN; ++jj) rv[jj] = (n0 + jj < NC) ? rhs[l * NCP + n0 + jj] : 0.f;
  #pragma unroll
                for (int i = 0; i < TM; ++i)
  #pragma unroll
                  for (int jj = 0; jj < TN; ++jj) acc[i][jj] = fmaf(dv[i], rv[jj], acc[i][jj]);
              }
  #pragma unroll
              for (int i = 0; i < TM; ++i)
  #pragma unroll
                for (int jj = 0; jj < TN; ++jj)
                  if (m0 + i < IB && n0 + jj < NC) {
                    sm.u.pc.y[(m0 + i) * NCP + n0 + jj] = acc[i][jj];
                    yg[(i0 + m0 + i) * NCP + n0 + jj] = acc[i][jj];
                  }
            }
          }
          __syncthreads();
          if (cown) {  // C (+/-)= V32_I^T Y_I
            const float sg = (pass == 1) ? 1.f : ((pass & 1) ? 1.f : -1.f);
  #pragma unroll 4
            for (int ii = 0; ii < IB; ++ii) {
              float vv[CM], yv[CN];
  #pragma unroll
              for (int i = 0; i < CM; ++i) vv[i] = (cm0 + i < NF) ? sg * sm.v32[(i0 + ii) * NCP + cm0 + i] : 0.f;
  #pragma unroll
              for (int j = 0; j < CN; ++j) yv[j] = (cn0 + j < NC) ? sm.u.pc.y[ii * NCP + cn0 + j] : 0.f;
  #pragma unroll
              for (int i = 0; i < CM; ++i)
  #pragma unroll
                for (int j = 0; j < CN; ++j) cacc[i][j] = fmaf(vv[i], yv[j], cacc[i][j]);
            }
          }
          __syncthreads();
        }
        if (pass == 1) {  // a-posteriori order control: 10 (|C| / |H0|)^2 <= 1e-12 -> order 1 suffices
          float cmax = 0.f, hmax = 0.f;
          if (cown)
  #pragma unroll
            for (int i = 0; i < CM; ++i)
  #pragma unroll
              for (int j = 0; j < CN; ++j)
                if (cm0 + i < NF && cn0 + j < NF) {
                  cmax = fmaxf(cmax, fabsf(cacc[i][j]));
                  hmax = fmaxf(hmax, fabsf(sm.v32[(NINT + cm0 + i) * NCP + cn0 + j]));
                }
          for (int o = 16; o > 0; o >>= 1) {
            cmax = fmaxf(cmax, __shfl_xor_sync(0xffffffffu, cmax, o));
            hmax = fmaxf(hmax, __shfl_xor_sync(0xffffffffu, hmax, o));
          }
          if ((tid & 31) == 0) {
            sm.red[tid >> 5] = cmax;
            sm.red[kThreads / 32 + (tid >> 5)] = hmax;
          }
          __syncthreads();
          if (tid == 0) {
            float cm = 0.f, hm = 0.f;
            for (int w = 0; w < kThreads / 32; ++w) {
              cm = fmaxf(cm, sm.red[w]);
              hm = fmaxf(hm, sm.red[kThreads / 32 + w]);
            }
            const double ratio = hm > 0.f ? static_cast<double>(cm) / hm : 0.0;
            bool ex = false;
            const int p = struct_order(ratio, A.p_max, A.eps32, ex);
            ex = ex || A.force_exact;
            sm.order = ex ? 1 : p;
            if (A.qlog && !use_tc) A.qlog[e] = static_cast<float>(ratio);
            if (ex) exact_push(A.xlist, A.xcount, e);  // (reached only for cells not yet rejected)
            sm.exact = ex ? 1 : 0;
          }
          __syncthreads();
          P = sm.order;
        }
        if (pass < P) {  // T = A0^-1 Y (Y in yg) -> behind Y in the scratch; rare path, fp64 accumulation
          float* tgl = yg + N * NCP;
          for (int idx = tid; idx < R * NC; idx += kThreads) {
            const int j = idx / NC, c = idx - j * NC;
            double acc = 0.0;
            for (int l = 0; l < N; ++l) acc = fma(__ldg(fx.X + l * R + j), static_cast<double>(yg[l * NCP + c]), acc);
            sm.u.pv.z[idx] = sm.s[j] * acc;
          }
          __syncthreads();
          for (int idx = tid; idx < N * NC; idx += kThreads) {
            const int i = idx / NC, c = idx - i * NC;
            double acc = 0.0;
            for (int l = 0; l < N; ++l)
              acc = fma(__ldg(fx.N0 + static_cast<int64_t>(i) * N + l), static_cast<double>(yg[l * NCP + c]), acc);
            for (int j = 0; j < R; ++j) acc = fma(__ldg(fx.X + i * R + j), sm.u.pv.z[j * NC + c], acc);
            tgl[i * NCP + c] = static_cast<float>(acc * ib);
          }
          __syncthreads();
        }
      }

      if (cown)
#pragma unroll
        for (int i = 0; i < CM; ++i)
#pragma unroll
          for (int j = 0; j < CN; ++j)
            if (cm0 + i < NF && cn0 + j < NC) sm.u.csm[(cm0 + i) * NCP + cn0 + j] = cacc[i][j];
      __syncthreads();
    }
    BIG_T(6);
    const bool cell_exact = sm.exact != 0;
    // ---------------------------------------------------------------- scatter
    // four entries per thread per pass: every load (vf, csm, the shared diagonal
    // blocks' partial sums) issued before the first store
    if constexpr (DPF % 2 == 0) {
      // even face dof counts: double2 work items, consecutive threads along one
      // (row, face block) run of DPF doubles (H rows start at multiples of DPF);
      // the g column after
      constexpr int H2 = DPF / 2, NIT = NF * NS * H2, SB2 = 5;
      for (int base = tid; base < NIT; base += SB2 * kThreads) {
        double2 val[SB2], old[SB2];
        double2* dst[SB2];
        bool acc[SB2];
#pragma unroll
        for (int u = 0; u < SB2; ++u) {
          const int idx = base + u * kThreads;
          dst[u] = nullptr;
          acc[u] = false;
          val[u] = make_double2(0.0, 0.0);
          if (idx >= NIT) continue;
          const int run = idx / H2, j2 = idx - run * H2;
          const int p = run / NS, qs = run - p * NS;
          const int ps = p / DPF, sub = p - ps * DPF;
          const int64_t rs = sm.rstart[ps];
          const int rk = sm.rank[ps * NS + qs];
          if (rs < 0 || rk < 0) continue;
          const int c = qs * DPF + 2 * j2;
          val[u] = make_double2(vf[p * NC + c] - static_cast<double>(sm.u.csm[p * NCP + c]),
                                vf[p * NC + c + 1] - static_cast<double>(sm.u.csm[p * NCP + c + 1]));
          if (cell_exact) val[u] = make_double2(0.0, 0.0);
          dst[u] = reinterpret_cast<double2*>(A.hval + rs + static_cast<int64_t>(sub) * sm.rlen[ps] + rk * DPF) + j2;
          acc[u] = parity == 1 && ps == qs;
        }
#pragma unroll
        for (int u = 0; u < SB2; ++u) old[u] = (dst[u] && acc[u]) ? *dst[u] : make_double2(0.0, 0.0);
#pragma unroll
        for (int u = 0; u < SB2; ++u)
          if (dst[u]) *dst[u] = acc[u] ? make_double2(old[u].x + val[u].x, old[u].y + val[u].y) : val[u];
      }
      for (int p = tid; p < NF; p += kThreads) {
        const int ps = p / DPF, sub = p - ps * DPF;
        if (sm.rstart[ps] < 0) continue;
        const double v = cell_exact ? 0.0 : vf[p * NC + NF] - static_cast<double>(sm.u.csm[p * NCP + NF]);
        double* gp = A.g + sm.grow[ps] + sub;
        *gp = parity ? *gp + v : v;
      }
    } else {
    constexpr int SB = 8;
    for (int base = tid; base < NF * NC; base += SB * kThreads) {
      double val[SB], old[SB];
      double* dst[SB];
      bool acc[SB];
#pragma unroll
      for (int u = 0; u < SB; ++u) {
        const int idx = base + u * kThreads;
        dst[u] = nullptr;
        acc[u] = false;
        val[u] = 0.0;
        if (idx >= NF * NC) continue;
        const int p = idx / NC, c = idx - p * NC;
        const int ps = p / DPF, sub = p - ps * DPF;
        const int64_t rs = sm.rstart[ps];
        if (rs < 0) continue;
        val[u] = cell_exact ? 0.0 : vf[p * NC + c] - static_cast<double>(sm.u.csm[p * NCP + c]);
        if (c == NF) {
          dst[u] = A.g + sm.grow[ps] + sub;
          acc[u] = parity != 0;
          continue;
        }
        const int qs = c / DPF, sj = c - qs * DPF;
        const int rk = sm.rank[ps * NS + qs];
        if (rk < 0) continue;
        dst[u] = A.hval + rs + static_cast<int64_t>(sub) * sm.rlen[ps] + rk * DPF + sj;
        acc[u] = parity == 1 && ps == qs;
      }
#pragma unroll
      for (int u = 0; u < SB; ++u) old[u] = (dst[u] && acc[u]) ? *dst[u] : 0.0;
#pragma unroll
      for (int u = 0; u < SB; ++u)
        if (dst[u]) *dst[u] = acc[u] ? old[u] + val[u] : val[u];
    }
    }
    __syncthreads();
    BIG_T(7);
#ifdef HDR_BIG_TIMING
    if (blockIdx.x == 0 && threadIdx.x == 0) g_big_prof[14] += 1;
    if (blockIdx.x == 0 && threadIdx.x == 0 && !tc_done) g_big_prof[15] += 1;
#endif
  }
  if (use_tc && (tid >> 5) == 0) umma::tmem_dealloc(sm.tmem, B::TCOLS);
}

template <int K>
void launch_big_t(const HybArgs& a, int parity, double* gws, const double* pre, int64_t grid, cudaStream_t st) {
  const size_t smem = sizeof(BigSmem<K>);
  cudaFuncSetAttribute(k_hyb_big<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  static const int use_tc = getenv("HDR_NO_TC") ? 0 : 1;  // HDR_NO_TC=1: CUDA-core correction (A/B timing)
  k_hyb_big<K><<<static_cast<unsigned>(grid), kThreads, smem, st>>>(a, parity, gws, use_tc, pre);
}

template <int K>
int64_t grid_big_t(const HybArgs& a) {
  const size_t smem = sizeof(BigSmem<K>);
  cudaFuncSetAttribute(k_hyb_big<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_hyb_big<K>, kThreads, smem);
  const int64_t cnt = parity_count(a.m);
  return std::max<int64_t>(1, std::min<int64_t>(cnt, static_cast<int64_t>(sms) * std::max(per_sm, 1)));
}

}  // namespace

#ifdef HDR_BIG_TIMING
extern "C" int hdr_debug_big_prof(unsigned long long* out) {
  cudaMemcpyFromSymbol(out, g_big_prof, sizeof(g_big_prof));  // 32 counters
  return 0;
}
#endif

bool hybridize_big_supported(int dim, int k) { return dim == 3 && (k == 2 || k == 3); }

int64_t hybridize_big_scratch_doubles(const HybArgs& a, int k) {
  if (k == 2) return grid_big_t<2>(a) * (big_scratch_doubles<2>() + static_cast<int64_t>(Big<2>::N) * Big<2>::NCP / 2 + 8);
  return grid_big_t<3>(a) * (big_scratch_doubles<3>() + static_cast<int64_t>(Big<3>::N) * Big<3>::NCP / 2 + 8);
}

void launch_hybridize_big(const HybArgs& a, int k, int parity, double* gws, const double* pre, cudaStream_t st) {
  if (k == 2) launch_big_t<2>(a, parity, gws, pre, grid_big_t<2>(a), st);
  else launch_big_t<3>(a, parity, gws, pre, grid_big_t<3>(a), st);
  count_launch();
}

}  // namespace hdr

// ---------------------------------------------------------------------------
// Per-cell products with fixed matrices, batched over all cells as one fp64
// GEMM before the element kernel: pre(:, e) = [N0 ; X^T] f_e (column-major,
// ld = N + R), on the fp64 tensor cores: a 128-thread CTA owns a 64 x 64 output
// tile (warp tiles of 32 x 32 = 4 x 4 DMMA m8n8k4 blocks); K staged in shared
// memory by 16, double-buffered, with row strides = 4 mod 16 so the fragment
// loads (8 rows x 4 k) hit every bank pair twice.
namespace hdr {
namespace {
constexpr int kGS = 68;  // shared row stride (doubles) of the staged tiles
__global__ void __launch_bounds__(128) k_gemm_f64_nn(int M, int Ncol, int Kd, const double* A, int lda,
                                                     const double* B, int ldb, double* C, int ldc) {
  __shared__ __align__(16) double As[2][16][kGS];  // As[k][m]
  __shared__ __align__(16) double Bs[2][16][kGS];  // Bs[k][n]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int m0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * 32;
  double d[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) d[i][j][0] = d[i][j][1] = 0.0;
  double ra[8], rb[8];  // the next chunk's tiles in flight (global -> registers) during this chunk's MMAs
  auto fetch = [&](int k0) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {  // 16 x 64 each: 1024 entries / 128 threads
      const int q = tid + u * 128;
      const int kk = q >> 6, mm = q & 63;  // A: k-major rows of 64 consecutive m
      ra[u] = (m0 + mm < M && k0 + kk < Kd) ? A[(m0 + mm) + static_cast<int64_t>(lda) * (k0 + kk)] : 0.0;
      const int nn = q >> 4, k2 = q & 15;  // B: column nn holds 16 consecutive k
      rb[u] = (n0 + nn < Ncol && k0 + k2 < Kd) ? B[(k0 + k2) + static_cast<int64_t>(ldb) * (n0 + nn)] : 0.0;
    }
  };
  auto stash = [&](int buf) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int q = tid + u * 128;
      As[buf][q >> 6][q & 63] = ra[u];
      Bs[buf][q & 15][q >> 4] = rb[u];
    }
  };
  fetch(0);
  stash(0);
  __syncthreads();
  const int nk = (Kd + 15) / 16;
  for (int c = 0; c < nk; ++c) {
    const int buf = c & 1;
    if (c + 1 < nk) fetch((c + 1) * 16);
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = As[buf][4 * ks + t][wm + 8 * i + g];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = Bs[buf][4 * ks + t][wn + 8 * j + g];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma_8x8x4(d[i][j][0], d[i][j][1], af[i], bf[j]);
    }
    if (c + 1 < nk) stash(buf ^ 1);
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int m = m0 + wm + 8 * i + g, n = n0 + wn + 8 * j + 2 * t + q;
        if (m < M && n < Ncol) C[m + static_cast<int64_t>(ldc) * n] = d[i][j][q];
      }
}
}  // namespace

void launch_gemm_f64_nn(int M, int Ncol, int Kd, const double* A, int lda, const double* B, int ldb, double* C,
                        int ldc, cudaStream_t st) {
  if (M <= 0 || Ncol <= 0) return;
  dim3 grid(static_cast<unsigned>((Ncol + 63) / 64), static_cast<unsigned>((M + 63) / 64));
  k_gemm_f64_nn<<<grid, 128, 0, st>>>(M, Ncol, Kd, A, lda, B, ldb, C, ldc);
  count_launch();
}
}  // namespace hdr
