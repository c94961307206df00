// Host side of the tcgen05 GEMM: TMA tensor maps, tile-size choice, launch.
#include "gemm.hpp"
#include "logits_tc.cuh"
#include "logits_tc2.cuh"

#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>
#include <string>

#include "errors.hpp"
#include "launch.cuh"

namespace mtg {

namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    MTG_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !p)
      fail(kCudaError, "cuTensorMapEncodeTiled entry point unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

CUtensorMap make_map(const void* ptr, int prec, int rows, int k_pad, int box_rows) {
  CUtensorMap m;
  const int elem = prec_elem_bytes(prec);
  CUtensorMapDataType dt = prec == kPrecI8     ? CU_TENSOR_MAP_DATA_TYPE_UINT8
                           : prec == kPrecBF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                               : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(k_pad), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(k_pad) * elem};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(128 / elem),
                       static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, dt, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    fail(kCudaError, "cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
  return m;
}

template <int PREC, int BN, int EPI, int FL = -1>
void launch_one(const GemmPlan& p, const GemmEpilogue& ep, cudaStream_t stream) {
  ensure_smem_attr(gemm_tc_kernel<PREC, BN, EPI, FL>, 227 * 1024);
  dim3 grid(p.n_tiles, p.m_tiles, p.splits);
  if (p.splits > 1) {  // split-K: the z splits of a tile form one cluster
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(kGemmThreads);
    cfg.dynamicSmemBytes = p.smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 1;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = p.splits;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    MTG_CUDA(cudaLaunchKernelEx(&cfg, gemm_tc_kernel<PREC, BN, EPI, FL>, p.a, p.b, p.a2, p.b2,
                                p.num_kb, p.nst, ep));
  } else {
    launch_k(gemm_tc_kernel<PREC, BN, EPI, FL>, grid, kGemmThreads, p.smem, stream, p.a, p.b,
             p.a2, p.b2, p.num_kb, p.nst, ep);
  }
  MTG_CUDA(cudaGetLastError());
}

template <int PREC>
void launch_prec(const GemmPlan& p, const GemmEpilogue& ep, cudaStream_t stream) {
  if (ep.part_m) {
    if (p.splits > 1) fail(kStateError, "gemm: softmax partials cannot be split over K");
    if (ep.bias || ep.residual || ep.relu || ep.d_step)
      fail(kStateError, "gemm: softmax-partials epilogue takes no bias/relu/residual");
    if (ep.part_ld % 4 != 0 || ep.part_ld * 32 < ep.N)
      fail(kStateError, "gemm: softmax partial pitch");
    switch (p.bn) {
      case 128: return launch_one<PREC, 128, kEpiSoftmaxParts>(p, ep, stream);
      case 256: return launch_one<PREC, 256, kEpiSoftmaxParts>(p, ep, stream);
    }
    fail(kStateError, "gemm: softmax partials need a 128/256-column tile");
  }
  if (ep.C_lo) {
    if constexpr (prec_is_tf32x3(PREC)) {
      switch (p.bn) {
        case 32: return launch_one<PREC, 32, kEpiTf32Out>(p, ep, stream);
        case 64: return launch_one<PREC, 64, kEpiTf32Out>(p, ep, stream);
        case 128: return launch_one<PREC, 128, kEpiTf32Out>(p, ep, stream);
        case 192: return launch_one<PREC, 192, kEpiTf32Out>(p, ep, stream);
        case 256: return launch_one<PREC, 256, kEpiTf32Out>(p, ep, stream);
      }
    }
    fail(kStateError, "gemm: TF32 operand output needs a TF32x3 GEMM");
  }
  if (ep.bf16_out) {
    if constexpr (PREC == kPrecBF16) {
      switch (p.bn) {
        case 32: return launch_one<PREC, 32, kEpiBf16Out>(p, ep, stream);
        case 64: return launch_one<PREC, 64, kEpiBf16Out>(p, ep, stream);
        case 128: return launch_one<PREC, 128, kEpiBf16Out>(p, ep, stream);
        case 192: return launch_one<PREC, 192, kEpiBf16Out>(p, ep, stream);
        case 256: return launch_one<PREC, 256, kEpiBf16Out>(p, ep, stream);
      }
    }
    fail(kStateError, "gemm: bf16 operand output needs a bf16 GEMM");
  }
  if (ep.seg_absmax) {
    if (ep.residual) fail(kStateError, "gemm: segment-max epilogue takes no residual");
    switch (p.bn) {
      case 32: return launch_one<PREC, 32, kEpiSegMax>(p, ep, stream);
      case 64: return launch_one<PREC, 64, kEpiSegMax>(p, ep, stream);
      case 128: return launch_one<PREC, 128, kEpiSegMax>(p, ep, stream);
      case 192: return launch_one<PREC, 192, kEpiSegMax>(p, ep, stream);
      case 256: return launch_one<PREC, 256, kEpiSegMax>(p, ep, stream);
    }
  }
  // The decoder GEMMs' options fixed at compile time (BN = 32; measured
  // +1.5 % int8; the same for the encoder's BN = 128 GEMMs was neutral).
  const int fl = (ep.bias ? 1 : 0) | (ep.relu ? 2 : 0) | (ep.residual ? 4 : 0) |
                 (ep.d_step ? 8 : 0);
  if (p.bn == 64 && fl == 5) return launch_one<PREC, 64, kEpiLinear, 5>(p, ep, stream);  // FFN-down
  // 64-column QKV at batch 64 (KV-cache slab offset only): the generic
  // variant spills for int8
  if (p.bn == 64 && fl == 8) return launch_one<PREC, 64, kEpiLinear, 8>(p, ep, stream);
  if (p.bn == 32) {
    switch (fl) {
      case 0: return launch_one<PREC, 32, kEpiLinear, 0>(p, ep, stream);
      case 3: return launch_one<PREC, 32, kEpiLinear, 3>(p, ep, stream);
      case 4: return launch_one<PREC, 32, kEpiLinear, 4>(p, ep, stream);
      case 5: return launch_one<PREC, 32, kEpiLinear, 5>(p, ep, stream);
      case 8: return launch_one<PREC, 32, kEpiLinear, 8>(p, ep, stream);
    }
  }
  switch (p.bn) {
    case 32: return launch_one<PREC, 32, kEpiLinear>(p, ep, stream);
    case 64: return launch_one<PREC, 64, kEpiLinear>(p, ep, stream);
    case 128: return launch_one<PREC, 128, kEpiLinear>(p, ep, stream);
    case 192: return launch_one<PREC, 192, kEpiLinear>(p, ep, stream);
    case 256: return launch_one<PREC, 256, kEpiLinear>(p, ep, stream);
  }
  fail(kStateError, "gemm: unsupported tile width");
}

__global__ void __launch_bounds__(kGemmThreads, 2) occupancy_probe_kernel(int* p) {
  extern __shared__ int probe_smem[];
  if (p) p[threadIdx.x] = probe_smem[threadIdx.x];
}

// CTAs of one split-K GEMM (cluster of `cs` along z, `smem` bytes each) that
// can be co-resident: clusters must fit inside one GPC, so e.g. at two CTAs
// per SM only 71 clusters of 4 (284 CTAs) fit, not 74 -- a 288-CTA grid then
// runs a second wave (measured: +10 us on the fp32 QKV GEMM). Cached per
// (device, smem, cs).
int max_cluster_ctas(int smem, int cs) {
  static std::mutex mu;
  static std::map<std::tuple<int, int, int>, int> cache;
  int dev = 0;
  MTG_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  const auto key = std::make_tuple(dev, smem, cs);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  // Queried with a stand-in of the GEMM's launch shape: for the tcgen05
  // kernels themselves the API reports one CTA per SM, while two run
  // (ncu: occupancy limited by shared memory at 2 blocks).
  auto k = occupancy_probe_kernel;
  ensure_smem_attr(k, 227 * 1024);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(1, 1, cs);
  cfg.blockDim = dim3(kGemmThreads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = cs;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, k, &cfg) != cudaSuccess) {
    cudaGetLastError();
    n = 0;
  }
  const int ctas = n * cs;
  cache[key] = ctas;
  if (std::getenv("MTG_PLAN_DEBUG")) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kGemmThreads, smem);
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, k);
    std::fprintf(stderr, "occupancy smem=%d cs=%d clusters=%d blocks/SM=%d regs=%d maxdyn=%d static=%zu\n",
                 smem, cs, n, per_sm, fa.numRegs, fa.maxDynamicSharedSizeBytes, fa.sharedSizeBytes);
  }
  return ctas;
}

}  // namespace

// Fewest m tiles for the long-K 64-column rule below (MTG_LONGK_MTILES A/B;
// measured: 3 -> decoder FFN-down at batch 64 f32 +3.1 %; 1 -> batch-1 p90 +4 %).
static const int kLongKMinMTiles = [] {
  const char* e = std::getenv("MTG_LONGK_MTILES");
  return e ? std::atoi(e) : 3;
}();

static const int kLongKBn = [] {
  const char* e = std::getenv("MTG_LONGK_BN");
  const int v = e ? std::atoi(e) : 64;
  return (v == 128 || v == 256) ? v : 64;
}();

GemmPlan plan_gemm(const Operand& a, const Operand& b, int m_max, int n, int force_bn,
                   int min_bn, bool allow_split) {
  const bool split_a = a.prec == kPrecTF32x3A && b.prec == kPrecTF32x3;  // plain fp32 A
  if ((a.prec != b.prec && !split_a) || a.k_pad != b.k_pad)
    fail(kShapeError, "gemm: operand precision / K mismatch");
  if (a.k_pad % (128 / prec_elem_bytes(a.prec)) != 0)
    fail(kShapeError, "gemm: K not padded to a 128-byte slab");
  GemmPlan p;
  p.prec = a.prec;
  p.num_kb = a.k_pad * prec_elem_bytes(a.prec) / 128;
  p.m_tiles = (m_max + 127) / 128;
  int bn = force_bn;
  if (!bn) {
    bn = 32;
    for (int cand : {256, 128, 64}) {
      if (p.m_tiles * ((n + cand - 1) / cand) >= 148) {
        bn = cand;
        break;
      }
    }
    // Several m tiles and a long fp32 K stream (the FFN-down GEMMs): 32-column
    // tiles re-read the hi+lo A rows once per tile; 64 columns with split-K
    // measured faster (fp32 encoder -6 %, decoder +3 % at batch 64; bf16 -0.2 %).
    if (bn == 32 && p.m_tiles >= kLongKMinMTiles && prec_is_tf32x3(b.prec) &&
        a.k_pad * prec_elem_bytes(a.prec) / 128 >= 32)
      bn = kLongKBn;
    bn = std::max(bn, min_bn);
  }
  // fp32 FFN-up at batch 64 (N = 4K, three m tiles): 64-column tiles, unsplit,
  // with the one-CTA-per-SM pipeline (more operand bytes in flight per CTA):
  // measured 16.5 -> 14.2 us per launch in the step graph (tools/step_trace.py).
  const bool ffn_up_deep = !force_bn && bn == 32 && prec_is_tf32x3(b.prec) && p.m_tiles >= 3 &&
                           n >= 4 * a.k_pad && a.k_pad >= 256;
  if (ffn_up_deep) bn = 64;
  // 128-column tiles just over one wave at one CTA per SM (the encoder's
  // fp32 QKV / FFN-up at batch 64: 156 / 208 tiles on 148 SMs, a second wave
  // of 8 / 60 tiles): 192-column tiles fit one wave (104 / 143 tiles).
  // Measured fp32 QKV 29.4 -> 19.7 us, FFN-up 35.9 -> 24.8 us; bf16 QKV
  // 8.8 -> 8.0 us (its FFN-up neutral); int8 slower (two CTAs per SM).
  {
    const int t128 = p.m_tiles * ((n + 127) / 128), t192 = p.m_tiles * ((n + 191) / 192);
    const bool fits = bn == 128 && t128 > 148 && t192 <= 148;
    if (!force_bn && fits &&
        (prec_is_tf32x3(b.prec) || (b.prec == kPrecBF16 && n % 192 == 0)))
      bn = 192;
  }
  // Just under one tile per SM at 32 columns (the fused QKV GEMM at batch 64:
  // 144 tiles, split 2): 64-column tiles split 3-4 ways read the activation
  // rows half as often (measured int8 5.2 -> 4.5 us, fp32 11.6 -> 11.2 us).
  if (!force_bn && !ffn_up_deep && bn == 32 && p.m_tiles >= 3 && p.m_tiles * ((n + 31) / 32) > 96 &&
      p.m_tiles * ((n + 31) / 32) < 148)
    bn = 64;
  p.bn = bn;
  p.n_tiles = (n + bn - 1) / bn;
  // Split-K over a z cluster when the output tiles cannot fill the SMs and a
  // tile's K stream is long (the DSMEM reduction costs ~1 us): aim for
  // >= ~160 KB of operand bytes per split, at most 8 (portable cluster).
  // MTG_SPLIT_CTAS / MTG_SPLIT_KB override the target grid size and bytes
  // per split (A/B experiments); default 160 KB per split.
  // Aim for two CTAs per SM (measured: fp32 p90 batch-1 -9 %, and with the
  // distributed split-K epilogue fp32 batch-64 +0.5 % over one per SM).
  static const int split_ctas_env = [] {
    const char* e = std::getenv("MTG_SPLIT_CTAS");
    return e ? std::atoi(e) : 0;
  }();
  // CTAs resident per SM with this tile (the pipeline-depth rule below).
  const int stage_b = gemm_stage_bytes(a.prec, bn);
  const int per_sm = (113 * 1024 - kGemmSmemExtra) / stage_b >= 2 ? 2 : 1;
  const int split_ctas = split_ctas_env > 0 ? split_ctas_env : 148 * per_sm;
  static const long long split_bytes = [] {
    const char* e = std::getenv("MTG_SPLIT_KB");
    return (e ? std::atoll(e) : 160LL) * 1024;
  }();
  const int tiles = p.m_tiles * p.n_tiles;
  const long long tile_bytes = static_cast<long long>(p.num_kb) * gemm_stage_bytes(a.prec, bn);
  const int by_bytes = static_cast<int>((tile_bytes + split_bytes - 1) / split_bytes);
  // MTG_GEMM_DEEP="NxK,..." (A/B): these shapes run unsplit with the deepest
  // one-CTA-per-SM pipeline.
  static const std::string deep_map = [] {
    const char* e = std::getenv("MTG_GEMM_DEEP");
    return std::string(e ? e : "");
  }();
  const bool deep = ffn_up_deep || (!deep_map.empty() && deep_map.find(std::to_string(n) + "x" +
                                                                      std::to_string(a.k_pad)) !=
                                                         std::string::npos);
  if (allow_split && !deep && tiles < 148 && p.num_kb >= 4 && by_bytes > 1)
    p.splits = std::max(1, std::min({p.num_kb / 2, split_ctas / tiles, kMaxSplits, by_bytes}));
  // Pipeline depth: no deeper than the K loop, and shallow enough for two
  // CTAs per SM when the tile allows it (epilogue / mainloop overlap, and the
  // next kernel's CTAs can start under PDL; measured: a one-CTA-per-SM depth
  // is slower even for single-wave grids).
  const int stage = gemm_stage_bytes(a.prec, bn);
  const int want = std::min(kMaxStages, std::max(2, p.num_kb));
  const int two_per_sm = (113 * 1024 - kGemmSmemExtra) / stage;
  const int one_per_sm = (227 * 1024 - kGemmSmemExtra) / stage;
  p.nst = std::min(want, two_per_sm >= 2 && !deep ? two_per_sm : one_per_sm);
  if (p.nst < 2 || p.nst * stage < kEpiStageBytes) fail(kStateError, "gemm: tile too large");
  if (p.splits > 1) {  // the parked split-K partial tile follows the epilogue staging
    const int need = kEpiStageBytes + 128 * (bn + 4) * 4;
    while (p.nst * stage < need && p.nst < one_per_sm) ++p.nst;
    if (p.nst * stage < need) p.splits = 1;
  }
  p.smem = p.nst * stage + kGemmSmemExtra;
  // One wave: fewer splits when the clusters would not all be co-resident.
  const int splits0 = p.splits;
  static const bool cluster_cap = [] {
    const char* e = std::getenv("MTG_CLUSTER_CAP");
    return !(e && e[0] == '0');
  }();
  while (cluster_cap && p.splits > 1 && tiles * p.splits > max_cluster_ctas(p.smem, p.splits))
    --p.splits;
  static const bool plan_debug = std::getenv("MTG_PLAN_DEBUG") != nullptr;
  if (plan_debug)
    std::fprintf(stderr, "plan n=%d k_pad=%d m=%d bn=%d tiles=%d splits=%d->%d nst=%d smem=%d cap=%d\n",
                 n, a.k_pad, m_max, bn, tiles, splits0, p.splits, p.nst, p.smem,
                 splits0 > 1 ? max_cluster_ctas(p.smem, splits0) : -1);
  p.a_box = (p.m_tiles == 1 && !split_a) ? std::max(8, (m_max + 7) / 8 * 8) : 128;
  p.a = make_map(a.ptr, a.prec, a.rows, a.k_pad, p.a_box);
  p.b = make_map(b.ptr, b.prec, b.rows, b.k_pad, bn);
  p.a2 = p.a;
  p.b2 = p.b;
  if (prec_is_tf32x3(b.prec)) {
    if (!b.ptr_lo) fail(kStateError, "gemm: TF32x3 needs the weight lo part");
    p.b2 = make_map(b.ptr_lo, b.prec, b.rows, b.k_pad, bn);
  }
  if (a.prec == kPrecTF32x3) {
    if (!a.ptr_lo) fail(kStateError, "gemm: TF32x3 needs the activation lo part");
    p.a2 = make_map(a.ptr_lo, a.prec, a.rows, a.k_pad, p.a_box);
  }
  return p;
}

namespace {
template <int PREC, int BN, int EG>
void launch_logits_one(const GemmPlan& p, const GemmEpilogue& ep, cudaStream_t stream) {
  ensure_smem_attr(logits_tc_kernel<PREC, BN, EG>, 227 * 1024);
  const int grid = std::min(148, p.m_tiles * p.n_tiles);
  launch_k(logits_tc_kernel<PREC, BN, EG>, grid, 64 + EG * 256, p.smem, stream, p.a, p.b, p.a2,
           p.b2, p.num_kb, p.nst, p.n_tiles, ep);
  MTG_CUDA(cudaGetLastError());
}
}  // namespace

GemmPlan plan_logits(const Operand& a, const Operand& b, int m_max, int n) {
  if (a.prec != b.prec || a.k_pad != b.k_pad)
    fail(kShapeError, "logits: operand precision / K mismatch");
  GemmPlan p;
  p.prec = a.prec;
  p.persistent = true;
  p.num_kb = a.k_pad * prec_elem_bytes(a.prec) / 128;
  p.m_tiles = (m_max + 127) / 128;
  p.bn = a.prec == kPrecTF32x3 ? 128 : 256;  // TF32x3 stages are twice as large
  p.n_tiles = (n + p.bn - 1) / p.bn;
  const int stage = gemm_stage_bytes(a.prec, p.bn);
  const int groups = a.prec == kPrecTF32x3 ? 1 : 2;  // must match launch_gemm's instantiation
  const int budget = 227 * 1024 - groups * kEpiStageBytes - kGemmSmemExtra;
  p.nst = std::min({kMaxStages, budget / stage, std::max(2, p.num_kb)});
  if (p.nst < 2) fail(kStateError, "logits: tile too large");
  p.smem = p.nst * stage + groups * kEpiStageBytes + kGemmSmemExtra;
  p.a_box = p.m_tiles == 1 ? std::max(8, (m_max + 7) / 8 * 8) : 128;
  p.a = make_map(a.ptr, a.prec, a.rows, a.k_pad, p.a_box);
  p.b = make_map(b.ptr, b.prec, b.rows, b.k_pad, p.bn);
  if (a.prec == kPrecTF32x3) {
    if (!a.ptr_lo || !b.ptr_lo) fail(kStateError, "logits: TF32x3 needs lo operands");
    p.a2 = make_map(a.ptr_lo, a.prec, a.rows, a.k_pad, p.a_box);
    p.b2 = make_map(b.ptr_lo, b.prec, b.rows, b.k_pad, p.bn);
  } else {
    p.a2 = p.a;
    p.b2 = p.b;
  }
  return p;
}

GemmPlan plan_logits_pair(const Operand& a, const Operand& b, int m_max, int n) {
  if (a.prec != kPrecTF32x3 || b.prec != kPrecTF32x3 || a.k_pad != b.k_pad)
    fail(kShapeError, "logits pair: TF32x3 operands with equal K");
  if (!a.ptr_lo || !b.ptr_lo) fail(kStateError, "logits pair: TF32x3 needs lo operands");
  GemmPlan p;
  p.prec = a.prec;
  p.persistent = true;
  p.pair = true;
  p.num_kb = a.k_pad * prec_elem_bytes(a.prec) / 128;
  p.m_tiles = (m_max + 255) / 256;
  p.bn = 256;
  p.n_tiles = (n + p.bn - 1) / p.bn;
  const int stage = 4 * 128 * 128;
  const int budget = 227 * 1024 - kEpiStageBytes - kGemmSmemExtra;
  p.nst = std::min({kMaxStages, budget / stage, std::max(2, p.num_kb)});
  if (p.nst < 2) fail(kStateError, "logits pair: tile too large");
  p.smem = p.nst * stage + kEpiStageBytes + kGemmSmemExtra;
  p.a_box = m_max <= 128 ? std::max(8, (m_max + 7) / 8 * 8) : 128;
  p.a = make_map(a.ptr, a.prec, a.rows, a.k_pad, p.a_box);
  p.a2 = make_map(a.ptr_lo, a.prec, a.rows, a.k_pad, p.a_box);
  p.b = make_map(b.ptr, b.prec, b.rows, b.k_pad, 128);  // each CTA loads half the tile
  p.b2 = make_map(b.ptr_lo, b.prec, b.rows, b.k_pad, 128);
  p.at = make_map(a.ptr, a.prec, a.rows, a.k_pad, 64);    // M = 128 pair tiles
  p.at2 = make_map(a.ptr_lo, a.prec, a.rows, a.k_pad, 64);
  return p;
}

static void launch_logits_pair(const GemmPlan& p, const GemmEpilogue& ep, cudaStream_t stream) {
  ensure_smem_attr(logits_tc2_kernel, 227 * 1024);
  if (!ep.part_m) fail(kStateError, "logits: softmax partial buffers missing");
  if (ep.part_ld % 4 != 0 || ep.part_ld * 32 < ep.N)
    fail(kStateError, "logits pair: softmax partial pitch");
  // Tiles go round-robin to the pairs, m fastest (the pair tiles sharing a
  // weight tile run together). With an even number of m tiles an odd pair
  // count alternates each pair between the full first m tile and the
  // partial last one instead of pinning half the pairs to the heavy tiles.
  int pairs = std::min(74, p.m_tiles * p.n_tiles);
  if (p.m_tiles % 2 == 0 && pairs % 2 == 0 && pairs > 1) --pairs;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * pairs);
  cfg.blockDim = dim3(320);
  cfg.dynamicSmemBytes = p.smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  MTG_CUDA(cudaLaunchKernelEx(&cfg, logits_tc2_kernel, p.a, p.b, p.a2, p.b2, p.at, p.at2,
                              p.num_kb, p.nst, p.n_tiles, ep));
  MTG_CUDA(cudaGetLastError());
}

void launch_gemm(const GemmPlan& p, const GemmEpilogue& ep_in, cudaStream_t stream) {
  GemmEpilogue ep = ep_in;
  ep.a_box = p.a_box;
  static const int split_dist = [] {
    const char* e = std::getenv("MTG_SPLITK_DIST");
    return e ? std::atoi(e) : 1;
  }();
  ep.split_dist = split_dist;
  if (p.pair) return launch_logits_pair(p, ep, stream);
  if (p.persistent) {
    if (!ep.part_m) fail(kStateError, "logits: softmax partial buffers missing");
    switch (p.prec) {
      case kPrecI8: return launch_logits_one<kPrecI8, 256, 2>(p, ep, stream);
      case kPrecBF16: return launch_logits_one<kPrecBF16, 256, 2>(p, ep, stream);
      case kPrecTF32x3: return launch_logits_one<kPrecTF32x3, 128, 1>(p, ep, stream);
    }
    fail(kStateError, "logits: unknown precision");
  }
  switch (p.prec) {
    case kPrecI8: return launch_prec<kPrecI8>(p, ep, stream);
    case kPrecBF16: return launch_prec<kPrecBF16>(p, ep, stream);
    case kPrecTF32x3: return launch_prec<kPrecTF32x3>(p, ep, stream);
    case kPrecTF32x3A: return launch_prec<kPrecTF32x3A>(p, ep, stream);
  }
  fail(kStateError, "gemm: unknown precision");
}

}  // namespace mtg
