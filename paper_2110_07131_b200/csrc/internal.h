// internal.h -- host-side declarations shared between the rmips translation units.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include "common.cuh"

#include <atomic>
#include <cstdlib>
#include <mutex>
#include <unordered_map>
#include <utility>

namespace rmips {

// Kernel launches issued by this library (own kernels + CUB device-sort kernels), for the
// bench's gpu_launches claim.  kCubSortKernels = kernels one CUB radix sort call launches
// (counted from the ncu launch list, profiles/).
extern std::atomic<long long> g_launches;
constexpr int kCubSortKernels = 10;  // histogram + exclusive-sum + 8 onesweep passes (64-bit keys)
inline void count_launch(int k = 1) { g_launches.fetch_add(k, std::memory_order_relaxed); }

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device, size): the call costs
// microseconds of host time, and query calls are short enough for that to show.
inline cudaError_t set_smem_attr(const void* func, int bytes) {
  static std::mutex mu;
  static std::unordered_map<const void*, int> done[16];
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  int& have = done[dev & 15][func];
  if (have >= bytes) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) have = bytes;
  return e;
}

// Scratch of one build call (owned by abi.cu, freed before rmips_build_index returns).
#define CK_PDL(x)                    \
  do {                               \
    const cudaError_t e_pdl_ = (x);  \
    if (e_pdl_ != cudaSuccess) return e_pdl_; \
  } while (0)
// Launch with programmatic stream serialisation (PDL): the kernel may start while its stream predecessor
// drains; it must call pdl_enter() (common.cuh) before reading anything the predecessor writes.
extern bool g_pdl;  // (on; the development library reads RMIPS_NO_PDL at every launch instead)
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
#ifdef RMIPS_DEV
  cfg.numAttrs = getenv("RMIPS_NO_PDL") ? 0 : 1;  // development: the chain without PDL
#else
  cfg.numAttrs = g_pdl ? 1 : 0;
#endif
  return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

struct BuildCtx {
  rmips_index_s* idx = nullptr;
  int64_t mb = 0;                 // items the lists are built over (idx->mprime)
  void* scratch_arena = nullptr;  // the single allocation of the build scratch below
  uint64_t* nkey = nullptr;       // [2][m + n] sort keys in/out: fp64 norm bits, top bit set for items
  int32_t* nval = nullptr;        // [2][m + n] sort values in/out: concatenated index (items first)
  int32_t* inv_u = nullptr;       // [n] original user row -> norm-sorted row
  unsigned int* maxabs = nullptr; // max |p_j| bits
  float* scale_dev = nullptr;     // 2^e
  void* cub_tmp = nullptr;
  size_t cub_bytes = 0;
  int32_t* cand = nullptr;        // [n][cstride] candidate item positions
  int cstride = kCand;            // candidate slots per row: 128, or 256 for k_max > kQ128MaxKmax
  int32_t* ccount = nullptr;      // [n] candidates per row, -1 = overflowed
  int32_t* ovf_list = nullptr;    // [n] overflowed rows
  int* ovf_count = nullptr;       // device counter
  unsigned long long* cand_total = nullptr;  // device: candidates kept by the filter (sum over rows)
  unsigned long long* tiles_done = nullptr;  // device: (128-user tile, item tile) contractions issued
};

// Regrouped tensor-core builds (build_tc2cta.cu): head-pass thetas -> rows sorted by theta -> U16 copy
struct Regroup {
  void* buf = nullptr;   // the one scratch allocation
  float* th = nullptr;   // [n] head-pass theta per index row
  float* ths = nullptr;  // [n] sorted (descending): theta per regrouped row
  int32_t* io = nullptr; // [n] iota
  int32_t* pm = nullptr; // [n] regrouped row -> index row
  void* cub = nullptr;
  size_t cub_bytes = 0;
  __half* U16b = nullptr;  // [n][ldh] U16 rows in regrouped order
  uint32_t* ent = nullptr; // [n][slots] head-pass candidate entries (index row order)
  uint4* meta = nullptr;   // [n] head-pass row state
};
cudaError_t regroup_alloc(Regroup& g, int64_t n, int ldh, int slots, cudaStream_t st);
cudaError_t regroup_rows(Regroup& g, const __half* U16, int64_t n, int ldh, cudaStream_t st);
void regroup_free(Regroup& g, cudaStream_t st);

size_t build_cub_bytes(int64_t n, int64_t m);
cudaError_t build_prep(BuildCtx& c, const float* Q, const float* P, cudaStream_t st);
cudaError_t build_simt(const BuildCtx& c, cudaStream_t st);
cudaError_t build_tc(const BuildCtx& c, cudaStream_t st);  // build_tc.cu; cudaErrorNotSupported if unusable
cudaError_t build_tcq(const BuildCtx& c, cudaStream_t st);  // build_tcq.cu (any d_pad)
cudaError_t build_tc2cta(const BuildCtx& c, cudaStream_t st);  // build_tc2cta.cu (CTA pairs, d_pad <= 256)
// Candidate slots per row the build will use (BuildCtx::cstride): 256 when k_max > kQ128MaxKmax and the
// positions fit the 4-byte entries (m <= 2^20), else 128.
constexpr int kQ128MaxKmax = 80;
int build_cand_stride(int kmax, int64_t mb, int build_flags, int d);
cudaError_t build_select(BuildCtx& c, cudaStream_t st);
cudaError_t build_fallback(BuildCtx& c, int nrows, double* scratch, int grid, cudaStream_t st);
cudaError_t build_blocks(BuildCtx& c, cudaStream_t st);

// Query workspace layout (carved from rmips_index_s::ws by abi.cu).
struct QueryCtx {
  rmips_index_s* idx = nullptr;
  const float* q = nullptr;      // [b][d] caller's queries (device)
  int b = 0, k = 0, flags = 0;
  int nsub = 0;                  // sub-batches of kQB queries
  // per sub-batch, sorted by norm descending (Alg. 3 line 1 computes ||q||)
  __half* Q16 = nullptr;         // [nsub][kQB][ldh] fp16 q*2^eq (sorted)
  float* qn = nullptr;           // [nsub][kQB] ||q|| rounded up (sorted; -1 padding)
  float* qerr = nullptr;         // [nsub][kQB] filter error bound, scaled units
  float* qscale = nullptr;       // [nsub] 2^eq
  int32_t* qperm = nullptr;      // [nsub][kQB] sorted slot -> input query index (-1 padding)
  int32_t* qcount = nullptr;     // [nsub] queries in the sub-batch
  double* qnrm = nullptr;        // [nsub][kQB] ||q|| in input order (query prep scratch)
  float* qcmax = nullptr;        // [nsub][kQB / 8] max |q_j| per prep CTA (query prep scratch)
  int32_t* wlen = nullptr;       // [nsub * nblocks] Lemma 3 prefix of every (sub-batch, user tile)
  // outputs of the filter
  unsigned long long* counters = nullptr;  // kNumCounters (+ accepted / undecided list sizes)
  uint64_t* acc = nullptr;       // accepted keys (q_input << 32 | original user id)
  uint32_t* bits = nullptr;      // or: accepted pairs as bits of a [b][nw] word matrix (no sort)
  int64_t nw = 0;                // words per query row of bits, ceil(n / 32)
  uint8_t* dirty = nullptr;      // [b][nbr] one byte per 32-word block of bits: set when a bit in it is
  int64_t nbr = 0;               // blocks per query row, ceil(nw / 32)
  uint64_t* und = nullptr;       // undecided (q_input << 32 | sorted user position)
  int32_t* scan_cnt = nullptr;   // [cap] P' index: items of P' that beat q, for the scan after P'
  uint64_t* scan_rec = nullptr;  // [cap] the pairs left for Alg. 2's scan, packed densely
  int32_t* scan_beats = nullptr; // [cap] ... with the count of items already known to beat q
  int64_t cap = 0;               // capacity of acc and of und
  int64_t sorted_n = 0;          // keys sorted by query_sort (reserved slots, sentinels last)
  uint64_t* acc_sorted = nullptr;  // (also holds the 32-bit packed keys of the fast output path)
  void* cub_tmp = nullptr;
  size_t cub_bytes = 0;
  int* flags_dev = nullptr;
  cudaEvent_t ev_k[2] = {nullptr, nullptr};  // (timing only) around the filter kernel itself
};

// TMA descriptor of a 2-D fp16 tensor [rows][cols], box box_rows x 64, SWIZZLE_128B (build_tc.cu).
bool make_tmap_f16_box(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows,
                       uint32_t box_cols = 64);
// Columns TMA loads for the LAST 64-column K block of a d-column row: the K steps of 16 that hold data
// (16 * ceil(d / 16) - 64 * (KB - 1)), rounded up to a box of 16, 32 or 64 columns (swizzle 32, 64 or
// 128 bytes).  d = 200: 16 columns, so a row streams 416 bytes instead of 512.
int tail_cols(int d);

cudaError_t query_prep(QueryCtx& c, cudaStream_t st);
cudaError_t query_filter_simt(QueryCtx& c, cudaStream_t st);
cudaError_t query_filter_tc(QueryCtx& c, cudaStream_t st);  // query_tc.cu
cudaError_t query_exact(QueryCtx& c, cudaStream_t st);
cudaError_t query_output(QueryCtx& c, int64_t* offsets, int32_t* user_ids, int64_t capacity, cudaStream_t st);
size_t query_cub_bytes(int64_t cap);
size_t query_scan_bytes(int64_t items);
int64_t query_bits_chunks(int b, int64_t nw);  // warp chunks of the bit-matrix output (scan items)
// zero four small regions (counts in 32-bit words, <= 128 each) in one launch (build.cu)
cudaError_t zero4(cudaStream_t st, void* a, int na, void* b, int nb, void* c, int nc, void* d, int nd);
cudaError_t query_sort(QueryCtx& c, int64_t total, int end_bit, cudaStream_t st);
// obase / obase_next (device words, both NULL for a single call): ids already written by earlier batches
// of rmips_query_batches; this batch's running total is stored to obase_next
// fold (batched calls): the batch's counters are folded into it (see k_bits_emit)
cudaError_t query_output_bits(QueryCtx& c, int64_t* offsets, int32_t* user_ids, int64_t capacity, cudaStream_t st,
                              const int64_t* obase = nullptr, int64_t* obase_next = nullptr,
                              unsigned long long* fold = nullptr);

}  // namespace rmips
