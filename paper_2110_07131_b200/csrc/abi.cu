// abi.cu -- the C ABI (include/rmips.h): validation, memory ownership, kernel orchestration.
// No exceptions cross the boundary; every CUDA error becomes RMIPS_ERR_CUDA with a message in
// rmips_last_error().  All work is enqueued on the caller's stream.
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "common.cuh"
#include "internal.h"

using namespace rmips;

std::atomic<long long> rmips::g_launches{0};
bool rmips::g_pdl = true;

namespace {

// CUDA-event phase timer (only when the caller asked for timing).  Events come from a per-thread
// pool (cudaEventCreate / Destroy per mark cost several microseconds of host time between the
// launches of a timed call).
thread_local std::vector<cudaEvent_t> g_ev_pool;
// Every mark also closes the previous NVTX range and opens the next phase's (names below), so an
// Nsight timeline shows the phases of each call; NVTX costs a pointer test when no tool is attached.
struct PhaseTimer {
  bool on = false;
  cudaStream_t st = nullptr;
  cudaEvent_t ev[8] = {};
  int n = 0;
  const char* const* names = nullptr;  // NVTX range opened by mark i (nullptr: none)
  bool open = false;
  PhaseTimer(bool enable, cudaStream_t s, const char* const* nm) : on(enable), st(s), names(nm) {}
  void mark() {
    if (open) nvtxRangePop();
    open = false;
    if (names && n < 8 && names[n]) {
      nvtxRangePushA(names[n]);
      open = true;
    }
    if (!on || n >= 8) {
      ++n;
      return;
    }
    if (!g_ev_pool.empty()) {
      ev[n] = g_ev_pool.back();
      g_ev_pool.pop_back();
    } else if (cudaEventCreate(&ev[n]) != cudaSuccess) {
      ev[n] = nullptr;
    }
    if (ev[n]) cudaEventRecord(ev[n], st);
    ++n;
  }
  double between(int a, int b) const {
    float ms = -1.f;
    if (!on || a >= n || b >= n || a >= 8 || b >= 8 || !ev[a] || !ev[b]) return -1.0;
    if (cudaEventElapsedTime(&ms, ev[a], ev[b]) != cudaSuccess) return -1.0;
    return ms;
  }
  ~PhaseTimer() {
    if (open) nvtxRangePop();
    for (int i = 0; i < n && i < 8; ++i)
      if (ev[i]) g_ev_pool.push_back(ev[i]);
  }
};
const char* const kBuildPhases[] = {"rmips_build: B1-B3 prep (norms, sort, convert)",
                                    "rmips_build: B4 contraction + candidate filter",
                                    "rmips_build: B5-B6 exact select, fallback, blocks", nullptr, nullptr,
                                    nullptr, nullptr, nullptr};
const char* const kQueryPhases[] = {"rmips_query: Q1 prep", "rmips_query: Q2-Q3 Lemma 3 + filter",
                                    "rmips_query: Q4-Q5 exact decide / scan (+ bit-matrix output)",
                                    "rmips_query: counters readback", "rmips_query: Q6 sorted-key output",
                                    nullptr, nullptr, nullptr};

thread_local std::string g_err;

// Two events around the query filter kernel itself (timing only): the roofline of k_query_tc is its own
// duration, without the host's launch gaps before it.
struct KernelEvents {
  cudaEvent_t ev[2] = {nullptr, nullptr};
  ~KernelEvents() {
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
  }
  bool get(cudaEvent_t (&out)[2]) {
    for (int i = 0; i < 2; ++i)
      if (!ev[i] && cudaEventCreate(&ev[i]) != cudaSuccess) return false;
    out[0] = ev[0], out[1] = ev[1];
    return true;
  }
};
thread_local KernelEvents g_kev;

rmips_status_t fail(rmips_status_t s, const std::string& msg) {
  g_err = msg;
  return s;
}

struct CudaFail {
  cudaError_t e;
  const char* what;
  int line;
};

#define CK(expr)                                                          \
  do {                                                                    \
    cudaError_t e_ = (expr);                                              \
    if (e_ != cudaSuccess) throw CudaFail{e_, #expr, __LINE__};           \
  } while (0)

rmips_status_t from_cuda(const CudaFail& f) {
  if (f.e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    return fail(RMIPS_ERR_OOM, std::string("out of device memory at ") + f.what);
  }
  char buf[512];
  snprintf(buf, sizeof buf, "CUDA error %d (%s) at abi.cu:%d: %s", (int)f.e, cudaGetErrorString(f.e), f.line, f.what);
  return fail(RMIPS_ERR_CUDA, buf);
}

template <typename T>
T* dalloc(int64_t count, cudaStream_t st) {
  void* p = nullptr;
  if (count <= 0) count = 1;
  CK(cudaMallocAsync(&p, (size_t)count * sizeof(T), st));
  return static_cast<T*>(p);
}

template <typename T>
void dfree(T*& p, cudaStream_t st) {
  if (p) cudaFreeAsync((void*)p, st);
  p = nullptr;
}

// One allocation carved into many arrays (256-byte aligned): one host API call instead of ~25.
struct Arena {
  size_t off = 0;
  template <typename T>
  size_t take(int64_t count) {
    const size_t o = off;
    if (count <= 0) count = 1;
    off += ((size_t)count * sizeof(T) + 255) / 256 * 256;
    return o;
  }
};

void retain_pool() {
  static bool done = false;
  if (done) return;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done = true;
}

// small pinned host staging buffer (per thread)
struct Pinned {
  void* p = nullptr;
  ~Pinned() { if (p) cudaFreeHost(p); }
  template <typename T>
  T* get() {
    if (!p) CK(cudaMallocHost(&p, 4096));
    return static_cast<T*>(p);
  }
};
thread_local Pinned g_pin;

void free_index_arrays(rmips_index_s* x, cudaStream_t st) {
  if (x->arena) cudaFreeAsync(x->arena, st);  // every index array lives in the arena
  x->arena = nullptr;
  if (x->list_arena) cudaFreeAsync(x->list_arena, st);
  x->list_arena = nullptr;
  x->perm_u = x->perm_p = nullptr;
  x->unorm = x->pnorm = nullptr;
  x->unu = x->perr = x->U32 = x->P32 = x->thr = x->tb = nullptr;
  x->U16 = x->P16 = nullptr;
  x->tau = nullptr;
  x->ids = nullptr;
  x->d_counters = nullptr;
  x->d_flags = nullptr;
  if (x->ws) cudaFreeAsync(x->ws, st);
  x->ws = nullptr;
  x->ws_bytes = 0;
}

int round_up(int v, int a) { return (v + a - 1) / a * a; }

int fallback_grid(int64_t m) {
  const int64_t cap = ((int64_t)256 << 20) / (8 * (m > 0 ? m : 1));
  return (int)(cap < 1 ? 1 : cap > 148 * 4 ? 148 * 4 : cap);
}

// NEXT-2 ("re-builds the data structures"): a query with k > k_max extends the
// index in place to k_max' = k.  The norm-sorted, converted operands are reused; only B4-B6 run
// again (contraction + candidate filter, exact select + fallback, block table) into new list
// arrays, stream-ordered, with no host synchronisation.
void extend_lists(rmips_index_s* x, int kmax_new, cudaStream_t st) {
  const int64_t n = x->n, m = x->m;
  if (n == 0) {  // no user lists to extend: every query answers the empty set
    x->kmax = kmax_new;
    return;
  }
  Arena la;
  const size_t o_tau = la.take<double>((int64_t)kmax_new * n), o_ids = la.take<int32_t>((int64_t)kmax_new * n),
               o_thr = la.take<float>((int64_t)kmax_new * n), o_tb = la.take<float>((int64_t)kmax_new * x->nlb);
  void* larena = nullptr;
  CK(cudaMallocAsync(&larena, la.off, st));
  BuildCtx c;
  c.idx = x;
  c.mb = x->mprime;
  c.cstride = build_cand_stride(kmax_new, c.mb, x->build_flags, x->d);
  const int fb_grid = fallback_grid(m);
  Arena sa;
  const size_t o_sc = sa.take<float>(4), o_cand = sa.take<int32_t>(n * c.cstride), o_cc = sa.take<int32_t>(n),
               o_ovl = sa.take<int32_t>(n), o_ovc = sa.take<int>(1), o_ct = sa.take<unsigned long long>(2),
               o_scr = sa.take<double>((int64_t)fb_grid * m);
  void* sarena = nullptr;
  try {
    CK(cudaMallocAsync(&sarena, sa.off, st));
  } catch (...) {
    cudaFreeAsync(larena, st);
    throw;
  }
  char* S = static_cast<char*>(sarena);
  c.scale_dev = reinterpret_cast<float*>(S + o_sc);
  c.cand = reinterpret_cast<int32_t*>(S + o_cand);
  c.ccount = reinterpret_cast<int32_t*>(S + o_cc);
  c.ovf_list = reinterpret_cast<int32_t*>(S + o_ovl);
  c.ovf_count = reinterpret_cast<int*>(S + o_ovc);
  c.cand_total = reinterpret_cast<unsigned long long*>(S + o_ct);
  c.tiles_done = c.cand_total + 1;
  double* scratch = reinterpret_cast<double*>(S + o_scr);
  c.scratch_arena = sarena;
  float* hs = g_pin.get<float>();
  hs[0] = x->pscale;
  CK(cudaMemcpyAsync(c.scale_dev, hs, sizeof(float), cudaMemcpyHostToDevice, st));
  CK(cudaMemsetAsync(c.ovf_count, 0, sizeof(int), st));
  CK(cudaMemsetAsync(c.cand_total, 0, 2 * sizeof(unsigned long long), st));
  char* L = static_cast<char*>(larena);
  double* old_tau = x->tau;
  int32_t* old_ids = x->ids;
  float *old_thr = x->thr, *old_tb = x->tb;
  const int old_kmax = x->kmax;
  x->tau = reinterpret_cast<double*>(L + o_tau);
  x->ids = reinterpret_cast<int32_t*>(L + o_ids);
  x->thr = reinterpret_cast<float*>(L + o_thr);
  x->tb = reinterpret_cast<float*>(L + o_tb);
  x->kmax = kmax_new;
  try {
    cudaError_t e = cudaErrorNotSupported;
    if (!(x->build_flags & RMIPS_BUILD_SIMT)) e = build_tc(c, st);
    if (e == cudaErrorNotSupported) {
      cudaGetLastError();
      c.cstride = kCand;  // the SIMT build's lists (cand.cuh)
      e = build_simt(c, st);
    }
    CK(e);
    CK(build_select(c, st));
    CK(build_fallback(c, 1, scratch, fb_grid, st));
    CK(build_blocks(c, st));
  } catch (...) {
    x->tau = old_tau, x->ids = old_ids, x->thr = old_thr, x->tb = old_tb, x->kmax = old_kmax;
    cudaFreeAsync(sarena, st);
    cudaFreeAsync(larena, st);
    throw;
  }
  cudaFreeAsync(sarena, st);
  if (x->list_arena) cudaFreeAsync(x->list_arena, st);  // (the first lists stay in the main arena)
  x->list_arena = larena;
  x->cand_total = -1;  // not read back (no host synchronisation)
  x->tiles_done = -1;
}

}  // namespace

extern "C" {

const char* rmips_version(void) { return "rmips-b200 0.1 (sm_100a)"; }
const char* rmips_last_error(void) { return g_err.c_str(); }

const char* rmips_status_string(rmips_status_t s) {
  switch (s) {
    case RMIPS_OK: return "ok";
    case RMIPS_ERR_INVALID: return "invalid argument";
    case RMIPS_ERR_NONFINITE: return "non-finite input value";
    case RMIPS_ERR_K_RANGE: return "k out of range (1 <= k <= k_max)";
    case RMIPS_ERR_CAPACITY: return "result capacity too small";
    case RMIPS_ERR_CUDA: return "CUDA error";
    case RMIPS_ERR_OOM: return "out of device memory";
  }
  return "unknown status";
}

rmips_status_t rmips_build_index_pprime(const float* Q, int64_t n, const float* P, int64_t m, int32_t d,
                                        int32_t k_max, int64_t m_prime, int32_t build_flags, void* cuda_stream,
                                        rmips_index_t* out) {
  if (!out) return fail(RMIPS_ERR_INVALID, "out is NULL");
  if (m_prime < 1) return fail(RMIPS_ERR_INVALID, "m_prime < 1");
  *out = nullptr;
  if (n < 0 || m < 1 || d < 1) return fail(RMIPS_ERR_INVALID, "need n >= 0, m >= 1, d >= 1");
  if (d > kMaxDim) return fail(RMIPS_ERR_INVALID, "d > 1024 is not supported");
  if (d > 256 && (build_flags & RMIPS_BUILD_SIMT))
    return fail(RMIPS_ERR_INVALID, "the SIMT (CUDA-core) build covers d <= 256; the tensor-core build any d");
  if (n >= (int64_t)1 << 31 || m >= (int64_t)1 << 31) return fail(RMIPS_ERR_INVALID, "n, m must be < 2^31");
  if ((n > 0 && !Q) || !P) return fail(RMIPS_ERR_INVALID, "NULL input matrix");
  if (k_max < 1) return fail(RMIPS_ERR_K_RANGE, "k_max < 1");
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  retain_pool();
  rmips_index_s* x = new rmips_index_s();
  x->n = n; x->m = m; x->d = d; x->kmax = k_max; x->build_flags = build_flags;
  x->mprime = m_prime < m ? m_prime : m;
  x->dpad = round_up(d, 64);
  x->ldh = round_up(d, 16);
  x->pd = round_up(d, 8);
  x->nblocks = (n + kTileU - 1) / kTileU;
  if (x->mprime < m) {  // P' index: blocks of ceil(log2 n) users (the paper's O(log n))
    int lg = 1;
    while (((int64_t)1 << lg) < n) ++lg;
    x->bsz = lg;
  }
  x->nlb = (n + x->bsz - 1) / x->bsz;
  x->c1 = filter_c1(x->dpad);
  x->c2 = filter_c2(x->dpad);
  cudaGetDevice(&x->device);
  BuildCtx c;
  c.idx = x;
  c.mb = x->mprime;
  double* scratch = nullptr;
  PhaseTimer tm((build_flags & RMIPS_BUILD_TIMING) != 0, st, kBuildPhases);
  try {
    // index arrays (kept) and build scratch (freed before return): two allocations
    Arena ia;
    const size_t o_flags = ia.take<int>(4), o_ctr = ia.take<unsigned long long>(kNumCounters + 4),
                 o_pu = ia.take<int32_t>(n), o_pp = ia.take<int32_t>(m), o_un = ia.take<double>(n),
                 o_unu = ia.take<float>(n), o_pn = ia.take<double>(m), o_perr = ia.take<float>(m),
                 o_u16 = ia.take<__half>(n * x->ldh), o_u32 = ia.take<float>(n * d),
                 o_p16 = ia.take<__half>(m * x->ldh), o_p32 = ia.take<float>(m * x->pd),
                 o_tau = ia.take<double>((int64_t)k_max * n), o_ids = ia.take<int32_t>((int64_t)k_max * n),
                 o_thr = ia.take<float>((int64_t)k_max * n), o_tb = ia.take<float>((int64_t)k_max * x->nlb);
    CK(cudaMallocAsync(&x->arena, ia.off, st));
    char* A = static_cast<char*>(x->arena);
    x->d_flags = reinterpret_cast<int*>(A + o_flags);
    x->d_counters = reinterpret_cast<unsigned long long*>(A + o_ctr);
    x->perm_u = reinterpret_cast<int32_t*>(A + o_pu);
    x->perm_p = reinterpret_cast<int32_t*>(A + o_pp);
    x->unorm = reinterpret_cast<double*>(A + o_un);
    x->unu = reinterpret_cast<float*>(A + o_unu);
    x->pnorm = reinterpret_cast<double*>(A + o_pn);
    x->perr = reinterpret_cast<float*>(A + o_perr);
    x->U16 = reinterpret_cast<__half*>(A + o_u16);
    x->U32 = reinterpret_cast<float*>(A + o_u32);
    x->P16 = reinterpret_cast<__half*>(A + o_p16);
    x->P32 = reinterpret_cast<float*>(A + o_p32);
    x->tau = reinterpret_cast<double*>(A + o_tau);
    x->ids = reinterpret_cast<int32_t*>(A + o_ids);
    x->thr = reinterpret_cast<float*>(A + o_thr);
    x->tb = reinterpret_cast<float*>(A + o_tb);
    Arena sa;
    c.cub_bytes = build_cub_bytes(n, m);
    // exact-fallback CTAs (each with m fp64 of scratch): up to 4 per SM, scratch <= 256 MB
    const int fb_grid = fallback_grid(m);
    const size_t o_key = sa.take<uint64_t>(2 * (m + n)), o_val = sa.take<int32_t>(2 * (m + n)), o_inv = sa.take<int32_t>(n),
                 o_max = sa.take<unsigned int>(4), o_cub = sa.take<unsigned char>((int64_t)c.cub_bytes),
                 o_cand = sa.take<int32_t>(n * build_cand_stride(k_max, x->mprime, build_flags, d)),
                 o_cc = sa.take<int32_t>(n), o_ovl = sa.take<int32_t>(n),
                 o_ovc = sa.take<int>(1), o_ct = sa.take<unsigned long long>(2),
                 o_scr = sa.take<double>((int64_t)fb_grid * m);
    void* sarena = nullptr;
    CK(cudaMallocAsync(&sarena, sa.off, st));
    char* S = static_cast<char*>(sarena);
    c.nkey = reinterpret_cast<uint64_t*>(S + o_key);
    c.nval = reinterpret_cast<int32_t*>(S + o_val);
    c.inv_u = reinterpret_cast<int32_t*>(S + o_inv);
    c.maxabs = reinterpret_cast<unsigned int*>(S + o_max);
    c.scale_dev = reinterpret_cast<float*>(c.maxabs + 2);
    c.cub_tmp = S + o_cub;
    c.cand = reinterpret_cast<int32_t*>(S + o_cand);
    c.cstride = build_cand_stride(k_max, x->mprime, build_flags, d);
    c.ccount = reinterpret_cast<int32_t*>(S + o_cc);
    c.ovf_list = reinterpret_cast<int32_t*>(S + o_ovl);
    c.ovf_count = reinterpret_cast<int*>(S + o_ovc);
    c.cand_total = reinterpret_cast<unsigned long long*>(S + o_ct);
    c.tiles_done = c.cand_total + 1;
    scratch = reinterpret_cast<double*>(S + o_scr);
    c.scratch_arena = sarena;
    CK(zero4(st, c.cand_total, 4, x->d_flags, 4, c.maxabs, 4, c.ovf_count, 1));

    const long long l0 = g_launches.load();
    tm.mark();  // 0
    CK(build_prep(c, Q, P, st));
    tm.mark();  // 1
    if (n > 0) {
      cudaError_t e = cudaErrorNotSupported;
      if (!(build_flags & RMIPS_BUILD_SIMT)) e = build_tc(c, st);
      if (e == cudaErrorNotSupported) {
        cudaGetLastError();
        x->build_flags |= RMIPS_BUILD_SIMT;
        c.cstride = kCand;  // the SIMT build's lists (cand.cuh)
        e = build_simt(c, st);
      }
      CK(e);
      tm.mark();  // 2
      CK(build_select(c, st));
      CK(build_fallback(c, 1, scratch, fb_grid, st));  // no-op unless rows overflowed (device count)
      CK(build_blocks(c, st));
    } else {
      tm.mark();
    }
    tm.mark();  // 3
    x->phase_ms[14] = (double)(g_launches.load() - l0);
    int* hp = g_pin.get<int>();
    CK(cudaMemcpyAsync(hp, x->d_flags, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hp + 1, c.ovf_count, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hp + 2, c.scale_dev, sizeof(float), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hp + 4, c.cand_total, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    cudaFreeAsync(c.scratch_arena, st);
    c.scratch_arena = nullptr;
    CK(cudaStreamSynchronize(st));
    int flags = hp[0];
    x->overflow_rows = hp[1];
    memcpy(&x->cand_total, hp + 4, sizeof(int64_t));
    memcpy(&x->tiles_done, hp + 6, sizeof(int64_t));
    if (tm.on) {
      x->phase_ms[0] = tm.between(0, 1);
      x->phase_ms[1] = tm.between(1, 2);
      x->phase_ms[2] = tm.between(2, 3);
      x->phase_ms[3] = tm.between(0, 3);
    }
    memcpy(&x->pscale, hp + 2, sizeof(float));
    if (flags & kFlagNonfinite) {
      free_index_arrays(x, st);
      delete x;
      return fail(RMIPS_ERR_NONFINITE, "Q or P contains a NaN or Inf");
    }
  } catch (const CudaFail& f) {
    cudaStreamSynchronize(st);
    if (c.scratch_arena) cudaFreeAsync(c.scratch_arena, st);
    free_index_arrays(x, st);
    delete x;
    return from_cuda(f);
  }
  x->last_stream = st;
  *out = x;
  return RMIPS_OK;
}

rmips_status_t rmips_build_index_ex(const float* Q, int64_t n, const float* P, int64_t m, int32_t d, int32_t k_max,
                                    int32_t build_flags, void* cuda_stream, rmips_index_t* out) {
  return rmips_build_index_pprime(Q, n, P, m, d, k_max, m, build_flags, cuda_stream, out);
}

rmips_status_t rmips_build_index(const float* Q, int64_t n, const float* P, int64_t m, int32_t d, int32_t k_max,
                                 void* cuda_stream, rmips_index_t* out) {
  return rmips_build_index_ex(Q, n, P, m, d, k_max, RMIPS_BUILD_DEFAULT, cuda_stream, out);
}

rmips_status_t rmips_build_index_host(const float* Q, int64_t n, const float* P, int64_t m, int32_t d, int32_t k_max,
                                      void* cuda_stream, rmips_index_t* out) {
  if (!out) return fail(RMIPS_ERR_INVALID, "out is NULL");
  if (n < 0 || m < 1 || d < 1 || (n > 0 && !Q) || !P) return fail(RMIPS_ERR_INVALID, "bad sizes or NULL input");
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  float *dQ = nullptr, *dP = nullptr;
  rmips_status_t s;
  try {
    dQ = dalloc<float>(n * d, st);
    dP = dalloc<float>(m * d, st);
    if (n) CK(cudaMemcpyAsync(dQ, Q, (size_t)n * d * 4, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(dP, P, (size_t)m * d * 4, cudaMemcpyHostToDevice, st));
    s = rmips_build_index(n ? dQ : nullptr, n, dP, m, d, k_max, cuda_stream, out);
  } catch (const CudaFail& f) {
    s = from_cuda(f);
  }
  dfree(dQ, st);
  dfree(dP, st);
  return s;
}

constexpr size_t kBitsMaxBytes = (size_t)64 << 20;  // largest bit-matrix output (rmips.h)

static void ensure_ws(rmips_index_s* x, QueryCtx& c, int nsub, int64_t cap, cudaStream_t st) {
  const int ldh = x->ldh;
  // accepted pairs as a bit matrix when it is small enough (no key sort, no mid-call sync)
  const int64_t nw = (x->n + 31) / 32;
  const int64_t nch = query_bits_chunks(c.b, nw);  // its output pass keeps <= 3 nch int64 in acc_sorted's space
  if (cap < 3 * nch) cap = 3 * nch;  // (the output pass's counts, in-CTA offsets and CTA totals)
  size_t qcub = query_cub_bytes(cap);
  const size_t qscan = query_scan_bytes(nch);
  if (qscan > qcub) qcub = qscan;
  const bool use_bits = x->n > 0 && !(c.flags & RMIPS_FLAG_KEY_SORT) && (size_t)c.b * (size_t)nw * 4 <= kBitsMaxBytes &&
                        c.b <= cap;
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off += (bytes + 255) / 256 * 256; return o; };
  size_t oQ16 = take((size_t)nsub * kQB * ldh * 2), oqn = take((size_t)nsub * kQB * 4),
         oqe = take((size_t)nsub * kQB * 4), oqs = take((size_t)nsub * 4), oqp = take((size_t)nsub * kQB * 4),
         oqc = take((size_t)nsub * 4), oqnr = take((size_t)nsub * kQB * 8), oqcm = take((size_t)nsub * kQB / 8 * 4),
         owl = take((size_t)nsub * x->nblocks * 4), oacc = take((size_t)cap * 8),
         ound = take((size_t)cap * 8), oscn = take((size_t)cap * 4),
         osrec = take((size_t)cap * 8), osbt = take((size_t)cap * 4),
         osrt = take((size_t)cap * 8), ocub = take(qcub),
         obits = take(use_bits ? (size_t)c.b * nw * 4 + (size_t)c.b * ((nw + 31) / 32) : 0);  // + dirty bytes
  if (off > x->ws_bytes) {
    x->bits_len = 0;
    if (x->ws) cudaFreeAsync(x->ws, st);
    x->ws = nullptr;
    CK(cudaMallocAsync(&x->ws, off, st));
    x->ws_bytes = off;
  }
  char* b = static_cast<char*>(x->ws);
  c.Q16 = reinterpret_cast<__half*>(b + oQ16);
  c.qn = reinterpret_cast<float*>(b + oqn);
  c.qerr = reinterpret_cast<float*>(b + oqe);
  c.qscale = reinterpret_cast<float*>(b + oqs);
  c.qperm = reinterpret_cast<int32_t*>(b + oqp);
  c.qcount = reinterpret_cast<int32_t*>(b + oqc);
  c.qnrm = reinterpret_cast<double*>(b + oqnr);
  c.qcmax = reinterpret_cast<float*>(b + oqcm);
  c.wlen = reinterpret_cast<int32_t*>(b + owl);
  c.acc = reinterpret_cast<uint64_t*>(b + oacc);
  c.und = reinterpret_cast<uint64_t*>(b + ound);
  c.scan_cnt = reinterpret_cast<int32_t*>(b + oscn);
  c.scan_rec = reinterpret_cast<uint64_t*>(b + osrec);
  c.scan_beats = reinterpret_cast<int32_t*>(b + osbt);
  c.acc_sorted = reinterpret_cast<uint64_t*>(b + osrt);
  c.cub_tmp = b + ocub;
  c.bits = use_bits ? reinterpret_cast<uint32_t*>(b + obits) : nullptr;
  c.nw = nw;
  c.nbr = (nw + 31) / 32;
  c.dirty = use_bits ? reinterpret_cast<uint8_t*>(c.bits + (size_t)c.b * nw) : nullptr;
  // the matrix is left all zero by every completed query (k_bits_emit clears what it reads); it
  // is cleared here only when its place or size changed, or after a failed call
  const size_t nbits = use_bits ? (size_t)c.b * nw * 4 + (size_t)c.b * c.nbr : 0;  // words + dirty bytes
  if (!use_bits) x->bits_len = 0;  // this layout may write over the old matrix
  if (use_bits && (x->bits_off != obits || x->bits_len < nbits)) {
    CK(cudaMemsetAsync(c.bits, 0, nbits, st));
    x->bits_off = obits;
    x->bits_len = nbits;
  }
  c.cub_bytes = qcub;
  c.cap = cap;
  x->pair_cap = cap;
}

rmips_status_t rmips_query_ex(rmips_index_t idx, const float* q_batch, int32_t b, int32_t k, int32_t flags,
                              int64_t* offsets, int32_t* user_ids, int64_t capacity, int64_t* total_out,
                              void* cuda_stream) {
  if (!idx || !total_out) return fail(RMIPS_ERR_INVALID, "NULL index or total_out");
  if (b < 0 || capacity < 0) return fail(RMIPS_ERR_INVALID, "b < 0 or capacity < 0");
  if (b > 0 && (!q_batch || !offsets)) return fail(RMIPS_ERR_INVALID, "NULL q_batch or offsets");
  if (capacity > 0 && !user_ids) return fail(RMIPS_ERR_INVALID, "NULL user_ids with capacity > 0");
  if (k < 1) return fail(RMIPS_ERR_K_RANGE, "k < 1");
  if (k > idx->kmax && (flags & RMIPS_FLAG_NO_EXTEND)) return fail(RMIPS_ERR_K_RANGE, "k > k_max");
  if ((flags & RMIPS_FLAG_SIMT) && idx->d > 256)
    return fail(RMIPS_ERR_INVALID, "the SIMT (CUDA-core) query filter covers d <= 256; the tensor-core filter any d");
  if (flags & ~(RMIPS_FLAG_NO_EXTEND | RMIPS_FLAG_NO_BLOCKS | RMIPS_FLAG_VERIFY_SCAN | RMIPS_FLAG_FORCE_VERIFY | RMIPS_FLAG_SIMT | RMIPS_FLAG_TIMING |
                RMIPS_FLAG_KEY_SORT))
    return fail(RMIPS_ERR_INVALID, "unknown flag bits");
  rmips_index_s* x = idx;
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  x->last_stream = st;
  *total_out = 0;
  memset(&x->stats, 0, sizeof x->stats);
  x->stats.queries = b;
  if (b == 0) {
    if (offsets) {
      if (cudaMemsetAsync(offsets, 0, sizeof(int64_t), st) != cudaSuccess || cudaStreamSynchronize(st) != cudaSuccess)
        return fail(RMIPS_ERR_CUDA, "memset of offsets failed");
    }
    return RMIPS_OK;
  }
  try {
    if (k > x->kmax) extend_lists(x, k, st);  // NEXT-2: k_max' = k, in place
    QueryCtx c;
    c.idx = x; c.q = q_batch; c.b = b; c.k = k; c.flags = flags;
    // P' index (lists over the first mprime items): the lists only bound tau_k from below, so the
    // filter may reject (Lemma 1) but never accept; every other pair goes to the exact path
    if (x->mprime < x->m) c.flags |= RMIPS_FLAG_FORCE_VERIFY;
    c.nsub = (b + kQB - 1) / kQB;
    c.counters = x->d_counters;
    c.flags_dev = x->d_flags;
    int64_t cap = x->pair_cap > 0 ? x->pair_cap : (int64_t)1 << 20;
    unsigned long long* hc = g_pin.get<unsigned long long>();
    std::unique_ptr<PhaseTimer> tm;
    const long long l0 = g_launches.load();
    for (int attempt = 0; attempt < 3; ++attempt) {
      tm.reset(new PhaseTimer((flags & RMIPS_FLAG_TIMING) != 0, st, kQueryPhases));
      if (tm->on) g_kev.get(c.ev_k);
      ensure_ws(x, c, c.nsub, cap, st);
      tm->mark();  // 0
      static_assert(2 * (kNumCounters + 4) <= 128, "zero4 region");
      CK(zero4(st, x->d_counters, 2 * (kNumCounters + 4), x->d_flags, 4, nullptr, 0, nullptr, 0));
      CK(query_prep(c, st));
      tm->mark();  // 1
      if (x->n > 0) {
        cudaError_t e = cudaErrorNotSupported;
        if (!(flags & RMIPS_FLAG_SIMT) && !(x->build_flags & RMIPS_BUILD_SIMT)) e = query_filter_tc(c, st);
        x->stats.filter_kernel = (e != cudaErrorNotSupported);
        if (e == cudaErrorNotSupported) {
          cudaGetLastError();
          e = query_filter_simt(c, st);
        }
        CK(e);
        tm->mark();  // 2
        CK(query_exact(c, st));
        if (c.bits) CK(query_output_bits(c, offsets, user_ids, capacity, st));  // before the sync
      } else {
        tm->mark();
      }
      tm->mark();  // 3
      CK(cudaMemcpyAsync(hc, x->d_counters, sizeof(unsigned long long) * kNumCounters, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(reinterpret_cast<int*>(hc + kNumCounters), x->d_flags, sizeof(int), cudaMemcpyDeviceToHost,
                         st));
      CK(cudaStreamSynchronize(st));
      int fl = *reinterpret_cast<int*>(hc + kNumCounters);
      if (fl & kFlagNonfinite) return fail(RMIPS_ERR_NONFINITE, "query vector contains a NaN or Inf");
      unsigned long long need = hc[C_ACCEPTED_TOTAL] > hc[C_UND_TOTAL] ? hc[C_ACCEPTED_TOTAL] : hc[C_UND_TOTAL];
      if ((int64_t)need <= cap) break;
      cap = (int64_t)(need + need / 4 + 1024);
      if (attempt == 2) return fail(RMIPS_ERR_CUDA, "pair workspace did not converge");
    }
    rmips_stats_t& S = x->stats;
    S.queries = b;
    S.block_query_pairs = hc[C_BLOCK_PAIRS];
    S.block_query_pruned = hc[C_BLOCK_PRUNED];
    S.pairs_scored = hc[C_SCORED];
    S.pairs_rejected = hc[C_REJECTED];
    S.pairs_accepted_fast = hc[C_ACCEPT_FAST];
    S.pairs_undecided = hc[C_UNDECIDED];
    S.pairs_exact_accepted = hc[C_EXACT_ACCEPT];
    S.scans = hc[C_SCANS];
    S.items_scanned = hc[C_ITEMS_SCANNED];
    S.result_total = hc[C_ACC_REAL];
    S.tiles_scored = hc[C_TILES_SCORED];
    S.scan_exact = hc[C_SCAN_EXACT];
    const int64_t total = S.result_total;
    const int64_t reserved = (int64_t)hc[C_ACCEPTED_TOTAL];  // >= total: sentinel padding sorts last
    tm->mark();  // 4
    if (!c.bits) {
      CK(query_sort(c, reserved, 64, st));
      CK(query_output(c, offsets, user_ids, capacity, st));
      tm->mark();  // 5
      CK(cudaStreamSynchronize(st));
    } else {
      // bit-matrix output: offsets and ids were enqueued before the one synchronisation above
      tm->mark();  // 5
      if (tm->on) CK(cudaStreamSynchronize(st));  // (only for the phase timer's last events)
    }
    x->phase_ms[15] = (double)(g_launches.load() - l0);
    if (tm->on) {
      x->phase_ms[8] = tm->between(0, 1);
      x->phase_ms[9] = tm->between(1, 2);
      x->phase_ms[10] = tm->between(2, 3);
      x->phase_ms[11] = tm->between(4, 5);
      x->phase_ms[12] = tm->between(0, 5);
      float kms = -1.f;
      x->phase_ms[13] = (c.ev_k[0] && x->stats.filter_kernel && cudaEventElapsedTime(&kms, c.ev_k[0], c.ev_k[1]) == cudaSuccess)
                            ? kms : -1.0;
    }
    *total_out = total;
    if (total > capacity) return fail(RMIPS_ERR_CAPACITY, "result ids exceed capacity");
  } catch (const CudaFail& f) {
    cudaStreamSynchronize(st);
    x->bits_len = 0;
    return from_cuda(f);
  }
  return RMIPS_OK;
}

// rmips_query_batches: per batch, the counters the host checks after a single call are folded on the
// device by k_bits_emit (sums; the largest pair-workspace need; the OR of the error flags), so the
// batches run back to back with one synchronisation at the end.
__global__ void k_shift_offsets(int64_t* __restrict__ off, int64_t cnt, int64_t base) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < cnt) off[i] += base;
}

static void fill_stats(rmips_index_s* x, const unsigned long long* hc, int64_t nq) {
  rmips_stats_t& S = x->stats;
  S.queries = nq;
  S.block_query_pairs = hc[C_BLOCK_PAIRS];
  S.block_query_pruned = hc[C_BLOCK_PRUNED];
  S.pairs_scored = hc[C_SCORED];
  S.pairs_rejected = hc[C_REJECTED];
  S.pairs_accepted_fast = hc[C_ACCEPT_FAST];
  S.pairs_undecided = hc[C_UNDECIDED];
  S.pairs_exact_accepted = hc[C_EXACT_ACCEPT];
  S.scans = hc[C_SCANS];
  S.items_scanned = hc[C_ITEMS_SCANNED];
  S.result_total = hc[C_ACC_REAL];
  S.tiles_scored = hc[C_TILES_SCORED];
  S.scan_exact = hc[C_SCAN_EXACT];
}

// Events of a timed rmips_query_batches: per batch, 4 phase marks + 2 around the filter kernel.
thread_local std::vector<cudaEvent_t> g_bev;
static cudaEvent_t* batch_events(size_t count) {
  while (g_bev.size() < count) {
    cudaEvent_t e = nullptr;
    if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
    g_bev.push_back(e);
  }
  return g_bev.data();
}

rmips_status_t rmips_query_batches(rmips_index_t idx, const float* q_all, int64_t nq, int32_t batch, int32_t k,
                                   int32_t flags, int64_t* offsets, int32_t* user_ids, int64_t capacity,
                                   int64_t* total_out, void* cuda_stream) {
  if (!idx || !total_out) return fail(RMIPS_ERR_INVALID, "NULL index or total_out");
  if (nq < 0 || batch < 1 || capacity < 0) return fail(RMIPS_ERR_INVALID, "nq < 0, batch < 1 or capacity < 0");
  if (nq > 0 && (!q_all || !offsets)) return fail(RMIPS_ERR_INVALID, "NULL q_all or offsets");
  if (capacity > 0 && !user_ids) return fail(RMIPS_ERR_INVALID, "NULL user_ids with capacity > 0");
  if (k < 1) return fail(RMIPS_ERR_K_RANGE, "k < 1");
  if (k > idx->kmax && (flags & RMIPS_FLAG_NO_EXTEND)) return fail(RMIPS_ERR_K_RANGE, "k > k_max");
  if ((flags & RMIPS_FLAG_SIMT) && idx->d > 256)
    return fail(RMIPS_ERR_INVALID, "the SIMT (CUDA-core) query filter covers d <= 256; the tensor-core filter any d");
  if (flags & ~(RMIPS_FLAG_NO_EXTEND | RMIPS_FLAG_NO_BLOCKS | RMIPS_FLAG_VERIFY_SCAN | RMIPS_FLAG_FORCE_VERIFY |
                RMIPS_FLAG_SIMT | RMIPS_FLAG_TIMING | RMIPS_FLAG_KEY_SORT))
    return fail(RMIPS_ERR_INVALID, "unknown flag bits");
  rmips_index_s* x = idx;
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  const int d = x->d;
  *total_out = 0;
  const int64_t nw = (x->n + 31) / 32;
  const bool bits_path = nq > 0 && x->n > 0 && !(flags & RMIPS_FLAG_KEY_SORT) && (size_t)batch * nw * 4 <= kBitsMaxBytes;
  if (!bits_path) {
    // one rmips_query_ex per batch (a host synchronisation each), offsets shifted to the running total
    int64_t base = 0;
    bool over = false;
    unsigned long long sums[kNumCounters] = {};
    for (int64_t b0 = 0; b0 < nq || (nq == 0 && b0 == 0); b0 += batch) {
      const int32_t bt = (int32_t)(nq - b0 < batch ? nq - b0 : batch);
      int64_t t = 0;
      const int64_t room = over || base > capacity ? 0 : capacity - base;
      rmips_status_t s = rmips_query_ex(idx, bt ? q_all + b0 * d : nullptr, bt, k, flags, offsets + b0,
                                        room ? user_ids + base : nullptr, room, &t, cuda_stream);
      if (s == RMIPS_ERR_CAPACITY) over = true;
      else if (s != RMIPS_OK) return s;
      if (base && bt) {
        k_shift_offsets<<<(unsigned)((bt + 1 + 255) / 256), 256, 0, st>>>(offsets + b0, bt + 1, base);
        if (cudaGetLastError() != cudaSuccess) return fail(RMIPS_ERR_CUDA, "offset shift failed");
      }
      const rmips_stats_t& S = x->stats;
      sums[C_BLOCK_PAIRS] += S.block_query_pairs, sums[C_BLOCK_PRUNED] += S.block_query_pruned;
      sums[C_SCORED] += S.pairs_scored, sums[C_REJECTED] += S.pairs_rejected;
      sums[C_ACCEPT_FAST] += S.pairs_accepted_fast, sums[C_UNDECIDED] += S.pairs_undecided;
      sums[C_EXACT_ACCEPT] += S.pairs_exact_accepted, sums[C_SCANS] += S.scans;
      sums[C_ITEMS_SCANNED] += S.items_scanned, sums[C_ACC_REAL] += S.result_total;
      sums[C_TILES_SCORED] += S.tiles_scored, sums[C_SCAN_EXACT] += S.scan_exact;
      base += t;
      if (nq == 0) break;
    }
    if (cudaStreamSynchronize(st) != cudaSuccess) return fail(RMIPS_ERR_CUDA, "synchronisation failed");
    fill_stats(x, sums, nq);
    *total_out = base;
    return over || base > capacity ? fail(RMIPS_ERR_CAPACITY, "result ids exceed capacity") : RMIPS_OK;
  }
  x->last_stream = st;
  memset(&x->stats, 0, sizeof x->stats);
  unsigned long long* acc = nullptr;  // [kNumCounters] sums, [.] largest need, [.] flags OR, then run[2]
  try {
    if (k > x->kmax) extend_lists(x, k, st);
    const int64_t nb = (nq + batch - 1) / batch;
    const int nacc = kNumCounters + 2 + 2;
    acc = dalloc<unsigned long long>(nacc, st);
    int64_t* run = reinterpret_cast<int64_t*>(acc + kNumCounters + 2);  // running totals (ping-pong)
    int64_t cap = x->pair_cap > 0 ? x->pair_cap : (int64_t)1 << 20;
    unsigned long long* hc = g_pin.get<unsigned long long>();
    static_assert((kNumCounters + 4) * 8 <= 4096, "pinned staging");
    cudaEvent_t* E = (flags & RMIPS_FLAG_TIMING) ? batch_events((size_t)6 * nb) : nullptr;
    const long long l0 = g_launches.load();
    for (int attempt = 0;; ++attempt) {
      CK(cudaMemsetAsync(acc, 0, (size_t)nacc * 8, st));
      for (int64_t t = 0; t < nb; ++t) {
        if (E) CK(cudaEventRecord(E[6 * t], st));
        const int64_t b0 = t * batch;
        QueryCtx c;
        c.idx = x; c.q = q_all + b0 * d; c.b = (int)(nq - b0 < batch ? nq - b0 : batch); c.k = k; c.flags = flags;
        if (x->mprime < x->m) c.flags |= RMIPS_FLAG_FORCE_VERIFY;  // as rmips_query_ex
        c.nsub = (c.b + kQB - 1) / kQB;
        c.counters = x->d_counters;
        c.flags_dev = x->d_flags;
        if (E) c.ev_k[0] = E[6 * t + 4], c.ev_k[1] = E[6 * t + 5];
        ensure_ws(x, c, c.nsub, cap, st);
        if (!c.bits) throw CudaFail{cudaErrorUnknown, "bit-matrix workspace (always fits on this path)", __LINE__};
        CK(zero4(st, x->d_counters, 2 * (kNumCounters + 4), x->d_flags, 4, nullptr, 0, nullptr, 0));
        CK(query_prep(c, st));
        if (E) CK(cudaEventRecord(E[6 * t + 1], st));
        cudaError_t e = cudaErrorNotSupported;
        if (!(flags & RMIPS_FLAG_SIMT) && !(x->build_flags & RMIPS_BUILD_SIMT)) e = query_filter_tc(c, st);
        x->stats.filter_kernel = (e != cudaErrorNotSupported);
        if (e == cudaErrorNotSupported) {
          cudaGetLastError();
          e = query_filter_simt(c, st);
        }
        CK(e);
        if (E) CK(cudaEventRecord(E[6 * t + 2], st));
        CK(query_exact(c, st));
        CK(query_output_bits(c, offsets + b0, user_ids, capacity, st, run + (t & 1), run + ((t + 1) & 1), acc));
        if (E) CK(cudaEventRecord(E[6 * t + 3], st));
      }
      CK(cudaMemcpyAsync(hc, acc, (size_t)(kNumCounters + 2) * 8, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(hc + kNumCounters + 2, run + (nb & 1), 8, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      if (hc[kNumCounters + 1] & kFlagNonfinite) {
        dfree(acc, st);
        return fail(RMIPS_ERR_NONFINITE, "query vector contains a NaN or Inf");
      }
      const unsigned long long need = hc[kNumCounters];
      if ((int64_t)need <= cap) break;
      cap = (int64_t)(need + need / 4 + 1024);  // a batch outgrew the pair workspace: run them all again
      if (attempt == 2) {
        dfree(acc, st);
        return fail(RMIPS_ERR_CUDA, "pair workspace did not converge");
      }
    }
    fill_stats(x, hc, nq);
    x->phase_ms[15] = (double)(g_launches.load() - l0);
    if (E) {  // phase times summed over the batches (rmips_phase_times: ms[8..13])
      double ph[4] = {0, 0, 0, 0};
      float ms = 0.f;
      bool ok = true;
      for (int64_t t = 0; t < nb; ++t) {
        for (int i = 0; i < 3; ++i) {
          ok = ok && cudaEventElapsedTime(&ms, E[6 * t + i], E[6 * t + i + 1]) == cudaSuccess;
          ph[i] += ms;
        }
        if (x->stats.filter_kernel) {
          ok = ok && cudaEventElapsedTime(&ms, E[6 * t + 4], E[6 * t + 5]) == cudaSuccess;
          ph[3] += ms;
        }
      }
      ok = ok && cudaEventElapsedTime(&ms, E[0], E[6 * (nb - 1) + 3]) == cudaSuccess;
      x->phase_ms[8] = ok ? ph[0] : -1.0;
      x->phase_ms[9] = ok ? ph[1] : -1.0;
      x->phase_ms[10] = ok ? ph[2] : -1.0;
      x->phase_ms[11] = 0.0;
      x->phase_ms[12] = ok ? ms : -1.0;
      x->phase_ms[13] = ok && x->stats.filter_kernel ? ph[3] : -1.0;
    }
    const int64_t total = (int64_t)hc[kNumCounters + 2];
    dfree(acc, st);
    acc = nullptr;
    *total_out = total;
    if (total > capacity) return fail(RMIPS_ERR_CAPACITY, "result ids exceed capacity");
  } catch (const CudaFail& f) {
    cudaStreamSynchronize(st);
    x->bits_len = 0;
    if (acc) dfree(acc, st);
    return from_cuda(f);
  }
  return RMIPS_OK;
}

rmips_status_t rmips_query_batches_host(rmips_index_t idx, const float* q_all, int64_t nq, int32_t batch, int32_t k,
                                        int64_t* offsets, int32_t* user_ids, int64_t capacity, int64_t* total_out,
                                        void* cuda_stream) {
  if (!idx || !total_out) return fail(RMIPS_ERR_INVALID, "NULL index or total_out");
  if (nq < 0 || batch < 1 || capacity < 0) return fail(RMIPS_ERR_INVALID, "nq < 0, batch < 1 or capacity < 0");
  if (nq > 0 && (!q_all || !offsets)) return fail(RMIPS_ERR_INVALID, "NULL q_all or offsets");
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  float* dq = nullptr;
  int64_t* doff = nullptr;
  int32_t* dids = nullptr;
  rmips_status_t s;
  try {
    dq = dalloc<float>(nq * idx->d, st);
    doff = dalloc<int64_t>(nq + 1, st);
    dids = dalloc<int32_t>(capacity, st);
    if (nq) CK(cudaMemcpyAsync(dq, q_all, (size_t)nq * idx->d * 4, cudaMemcpyHostToDevice, st));
    s = rmips_query_batches(idx, dq, nq, batch, k, RMIPS_FLAG_NONE, doff, dids, capacity, total_out, cuda_stream);
    if (s == RMIPS_OK || s == RMIPS_ERR_CAPACITY) {
      CK(cudaMemcpyAsync(offsets, doff, (size_t)(nq + 1) * 8, cudaMemcpyDeviceToHost, st));
      if (s == RMIPS_OK && *total_out > 0)
        CK(cudaMemcpyAsync(user_ids, dids, (size_t)*total_out * 4, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
    }
  } catch (const CudaFail& f) {
    s = from_cuda(f);
  }
  dfree(dq, st); dfree(doff, st); dfree(dids, st);
  return s;
}

rmips_status_t rmips_query(rmips_index_t idx, const float* q_batch, int32_t b, int32_t k, int64_t* offsets,
                           int32_t* user_ids, int64_t capacity, int64_t* total_out, void* cuda_stream) {
  return rmips_query_ex(idx, q_batch, b, k, RMIPS_FLAG_NONE, offsets, user_ids, capacity, total_out, cuda_stream);
}

rmips_status_t rmips_query_host(rmips_index_t idx, const float* q_batch, int32_t b, int32_t k, int64_t* offsets,
                                int32_t* user_ids, int64_t capacity, int64_t* total_out, void* cuda_stream) {
  if (!idx || !total_out) return fail(RMIPS_ERR_INVALID, "NULL index or total_out");
  if (b < 0) return fail(RMIPS_ERR_INVALID, "b < 0");
  if (b > 0 && (!q_batch || !offsets)) return fail(RMIPS_ERR_INVALID, "NULL q_batch or offsets");
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  float* dq = nullptr;
  int64_t* doff = nullptr;
  int32_t* dids = nullptr;
  rmips_status_t s;
  try {
    dq = dalloc<float>((int64_t)b * idx->d, st);
    doff = dalloc<int64_t>((int64_t)b + 1, st);
    dids = dalloc<int32_t>(capacity, st);
    if (b) CK(cudaMemcpyAsync(dq, q_batch, (size_t)b * idx->d * 4, cudaMemcpyHostToDevice, st));
    s = rmips_query(idx, dq, b, k, doff, dids, capacity, total_out, cuda_stream);
    if (s == RMIPS_OK || s == RMIPS_ERR_CAPACITY) {
      if (b) CK(cudaMemcpyAsync(offsets, doff, (size_t)(b + 1) * 8, cudaMemcpyDeviceToHost, st));
      if (s == RMIPS_OK && *total_out > 0)
        CK(cudaMemcpyAsync(user_ids, dids, (size_t)*total_out * 4, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
    }
  } catch (const CudaFail& f) {
    s = from_cuda(f);
  }
  dfree(dq, st); dfree(doff, st); dfree(dids, st);
  return s;
}

rmips_status_t rmips_phase_times(rmips_index_t idx, double ms[16]) {
  if (!idx || !ms) return fail(RMIPS_ERR_INVALID, "NULL argument");
  for (int i = 0; i < 16; ++i) ms[i] = idx->phase_ms[i];
  return RMIPS_OK;
}

rmips_status_t rmips_query_stats(rmips_index_t idx, rmips_stats_t* out) {
  if (!idx || !out) return fail(RMIPS_ERR_INVALID, "NULL argument");
  *out = idx->stats;
  return RMIPS_OK;
}

rmips_status_t rmips_index_info(rmips_index_t idx, int64_t info[16]) {
  if (!idx || !info) return fail(RMIPS_ERR_INVALID, "NULL argument");
  for (int i = 8; i < 16; ++i) info[i] = 0;
  info[8] = idx->cand_total;
  info[9] = idx->tiles_done;
  info[10] = idx->mprime;
  info[11] = idx->build_kernel;
  info[12] = idx->cand_slots;
  info[0] = idx->n; info[1] = idx->m; info[2] = idx->d; info[3] = idx->kmax;
  info[4] = idx->dpad; info[5] = idx->bsz; info[6] = idx->overflow_rows; info[7] = idx->build_flags;
  return RMIPS_OK;
}

rmips_status_t rmips_index_export(rmips_index_t idx, int64_t* perm_u, int64_t* perm_p, double* tau, int32_t* ids) {
  if (!idx) return fail(RMIPS_ERR_INVALID, "NULL index");
  rmips_index_s* x = idx;
  const int64_t n = x->n, m = x->m, K = x->kmax;
  try {
    std::vector<int32_t> pu(n > 0 ? n : 1), pp(m);
    if (n) CK(cudaMemcpy(pu.data(), x->perm_u, n * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(pp.data(), x->perm_p, m * 4, cudaMemcpyDeviceToHost));
    if (perm_u) for (int64_t i = 0; i < n; ++i) perm_u[i] = pu[i];
    if (perm_p) for (int64_t i = 0; i < m; ++i) perm_p[i] = pp[i];
    if ((tau || ids) && n) {
      std::vector<double> t(K * n);
      std::vector<int32_t> d(K * n);
      CK(cudaMemcpy(t.data(), x->tau, K * n * 8, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(d.data(), x->ids, K * n * 4, cudaMemcpyDeviceToHost));
      for (int64_t j = 0; j < K; ++j)
        for (int64_t r = 0; r < n; ++r) {
          if (tau) tau[j * n + pu[r]] = t[j * n + r];
          if (ids) ids[j * n + pu[r]] = d[j * n + r];
        }
    }
  } catch (const CudaFail& f) {
    return from_cuda(f);
  }
  return RMIPS_OK;
}

void rmips_free_index(rmips_index_t idx) {
  if (!idx) return;
  // stream-ordered after the index's last call (no host synchronisation)
  free_index_arrays(idx, idx->last_stream);
  delete idx;
}

}  // extern "C"
