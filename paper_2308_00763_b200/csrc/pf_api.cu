// pf_api.cu -- C ABI (include/pf_b200.h) over the sm_100a kernels.
//
// Host-side responsibilities only: argument validation with the reference's
// error semantics (filter.py:137-143 _validate_k, 55-60 from_name), buffer
// ownership, launch sequencing on the handle's stream, CUDA-graph replay of
// the per-frame launch pair, event timing.  Every arithmetic step of the
// tracking path runs on the device; there is no host compute path.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdio>
#include <string>
#include <vector>

#include "../../include/pf_b200.h"
#include "pf_kernels.cuh"
#include "pf_fused_sel.cuh"
#include "pf_philox.cuh"
#include "pf_staged.cuh"
#include "pf_video.cuh"
// host copies of the ziggurat tables
#undef PF_ZIG_QUAL
#define PF_ZIG_QUAL static const
#define PF_ZIG_KI PF_ZIG_KI_HOST
#define PF_ZIG_WI_BITS PF_ZIG_WI_BITS_HOST
#define PF_ZIG_FI_BITS PF_ZIG_FI_BITS_HOST
#define PF_ZIG_TABLES_HOST_PASS
#include "ziggurat_tables_host.inc"
#undef PF_ZIG_KI
#undef PF_ZIG_WI_BITS
#undef PF_ZIG_FI_BITS


namespace {

thread_local std::string g_err;

#define PF_CUDA(call, H)                                                                  \
  do {                                                                                    \
    cudaError_t _e = (call);                                                              \
    if (_e != cudaSuccess) {                                                              \
      (H) = std::string("CUDA error ") + cudaGetErrorString(_e) + " at " #call;           \
      return PF_ECUDA;                                                                    \
    }                                                                                     \
  } while (0)

// ---- host binary16 (RNE from f64; halfnum._bits_from_f64, halfnum.py:87-114)
uint64_t rne_shift(uint64_t sig, int shift) {
  uint64_t rem = sig & ((1ULL << shift) - 1);
  uint64_t out = sig >> shift;
  uint64_t half = 1ULL << (shift - 1);
  if (rem > half || (rem == half && (out & 1))) out += 1;
  return out;
}
uint16_t f64_to_f16(double x) {
  uint64_t bits;
  std::memcpy(&bits, &x, 8);
  uint16_t sign = (uint16_t)((bits >> 48) & 0x8000);
  int exp = (int)((bits >> 52) & 0x7FF);
  uint64_t frac = bits & 0xFFFFFFFFFFFFFULL;
  if (exp == 0x7FF) return frac ? 0x7E00 : (uint16_t)(sign | 0x7C00);
  int e = exp - 1023;
  if (exp == 0 || e < -25) return sign;
  if (e >= 16) return (uint16_t)(sign | 0x7C00);
  uint64_t sig = (1ULL << 52) | frac;
  uint64_t half;
  if (e >= -14) {
    uint64_t rounded = rne_shift(sig, 42);
    half = ((uint64_t)(e + 15) << 10) + rounded - (1ULL << 10);
  } else {
    half = rne_shift(sig, 42 + (-14 - e));
  }
  if ((half & 0x7FFF) >= 0x7C00) return (uint16_t)(sign | 0x7C00);
  return (uint16_t)(sign | half);
}
double f16_to_f64(uint16_t h) {
  double sign = (h & 0x8000) ? -1.0 : 1.0;
  int e = (h >> 10) & 0x1F;
  int frac = h & 0x3FF;
  if (e == 0x1F) return frac ? NAN : sign * INFINITY;
  if (e == 0) return sign * std::ldexp((double)frac, -24);
  return sign * std::ldexp((double)(frac | 0x400), e - 25);
}
void build_exp16(uint16_t* out) {
  for (int h = 0; h < 65536; ++h) {
    double v = f16_to_f64((uint16_t)h);
    if (std::isnan(v))
      out[h] = 0x7E00;
    else
      out[h] = f64_to_f16(std::exp(v));
  }
}

// NumPy pairwise_sum plan over n elements: leaves (start, len) + ops
void pw_plan(long long start, long long n, std::vector<long long>& ls, std::vector<int>& ll, std::vector<int>& ops) {
  if (n <= 128) {
    ops.push_back((int)ls.size());
    ls.push_back(start);
    ll.push_back((int)n);
    return;
  }
  long long n2 = n / 2;
  n2 -= n2 % 8;
  pw_plan(start, n2, ls, ll, ops);
  pw_plan(start + n2, n - n2, ls, ll, ops);
  ops.push_back(-1);
}

bool g_jump_ready[64] = {false};
int init_device_tables(int dev, std::string& err) {
  if (dev < 0 || dev >= 64) {
    err = "bad device";
    return PF_EINVAL;
  }
  if (g_jump_ready[dev]) return PF_OK;
  static pfr::Affine host[pfr::kJumpDigits][256];
  for (int d = 0; d < pfr::kJumpDigits; ++d)
    for (int v = 0; v < 256; ++v) host[d][v] = pfr::affine_pow((uint64_t)v << (8 * d));
  PF_CUDA(cudaMemcpyToSymbol(pfr::kJump, host, sizeof(host)), err);
  g_jump_ready[dev] = true;
  return PF_OK;
}

int kmode_of(int precision) { return precision == PF_FP64 ? 0 : precision == PF_FP32 ? 1 : 2; }
size_t real_size(int km) { return km == 0 ? 8 : km == 1 ? 4 : 2; }

int next_pow2(long long v) {
  int p = 1;
  while (p < v) p <<= 1;
  return p;
}

}  // namespace

// Parallel generator of the reference's Philox stream (pf_philox.cuh): scratch
// sized for the largest draw seen, the stream state and its device position.
struct PhxGen {
  pfp::PhxStream s{};
  unsigned long long* P = nullptr;  // device word position
  int* status = nullptr;            // device: nonzero if a window ran short
  double* v = nullptr;
  int *L = nullptr, *exit0 = nullptr, *entry = nullptr, *count = nullptr, *exitb = nullptr, *bad = nullptr;
  long long* base = nullptr;
  double* u_scratch = nullptr;
  int cap_blk = 0;

  void release() {
    void* ps[] = {P, status, v, L, exit0, entry, count, exitb, bad, base, u_scratch};
    for (void* q : ps)
      if (q) cudaFree(q);
    *this = PhxGen{};
  }
  // state11 = NumPy Philox state: key[2], counter[4], buffer[4], buffer_pos
  int init(const uint64_t* state11, std::string& err) {
    s.key[0] = state11[0];
    s.key[1] = state11[1];
    for (int i = 0; i < 4; ++i) s.ctr[i] = state11[2 + i];
    for (int i = 0; i < 4; ++i) s.buf[i] = state11[6 + i];
    s.pos = (int)state11[10];
    if (s.pos < 0 || s.pos > 4) {
      err = "bad Philox buffer position";
      return PF_EINVAL;
    }
    if (!P) {
      PF_CUDA(cudaMalloc(&P, 8), err);
      PF_CUDA(cudaMalloc(&status, 4), err);
      PF_CUDA(cudaMalloc(&u_scratch, 8), err);
    }
    return rewind(nullptr, err);
  }
  int rewind(cudaStream_t st, std::string& err) {
    PF_CUDA(cudaMemsetAsync(P, 0, 8, st), err);
    PF_CUDA(cudaMemsetAsync(status, 0, 4, st), err);
    return PF_OK;
  }
  int reserve(long long n, std::string& err) {
    const int nb = pfp::window_blocks(n);
    if (nb <= cap_blk) return PF_OK;
    void* ps[] = {v, L, exit0, entry, count, exitb, bad, base};
    for (void* q : ps)
      if (q) cudaFree(q);
    const size_t W = (size_t)nb * pfp::kBlk;
    PF_CUDA(cudaMalloc(&v, W * 8), err);
    PF_CUDA(cudaMalloc(&L, W * 4), err);
    PF_CUDA(cudaMalloc(&exit0, nb * 4), err);
    PF_CUDA(cudaMalloc(&entry, nb * 4), err);
    PF_CUDA(cudaMalloc(&count, nb * 4), err);
    PF_CUDA(cudaMalloc(&exitb, nb * 4), err);
    PF_CUDA(cudaMalloc(&bad, nb * 4), err);
    PF_CUDA(cudaMalloc(&base, nb * 8), err);
    cap_blk = nb;
    return PF_OK;
  }
  // n normals into out (device) and, with u_out, the random() after them
  int draw(cudaStream_t st, long long n, double* out, double* u_out, std::string& err) {
    int rc = reserve(n, err);
    if (rc) return rc;
    pfp::GenArgs a{};
    a.s = s;
    a.P = P;
    a.n = n;
    a.nblk = pfp::window_blocks(n);
    a.v = v;
    a.L = L;
    a.exit0 = exit0;
    a.entry = entry;
    a.count = count;
    a.exitb = exitb;
    a.bad = bad;
    a.base = base;
    a.out = out;
    a.u_out = u_out ? u_out : u_scratch;
    a.status = status;
    a.take_uniform = u_out ? 1 : 0;
    pfp::phx_classify<<<a.nblk, pfp::kThreads, 0, st>>>(a);
    pfp::phx_resolve<<<a.nblk, pfp::kThreads, 0, st>>>(a);
    pfp::phx_scan<<<1, pfp::kThreads, 0, st>>>(a);
    pfp::phx_emit<<<a.nblk, pfp::kThreads, 0, st>>>(a);
    PF_CUDA(cudaGetLastError(), err);
    return PF_OK;
  }
  int uniforms(cudaStream_t st, long long m, double* out, std::string& err) {
    pfp::phx_uniforms<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(s, P, m, out);
    pfp::phx_advance<<<1, 1, 0, st>>>(P, m);
    PF_CUDA(cudaGetLastError(), err);
    return PF_OK;
  }
  int check(std::string& err) {  // after a synchronisation
    int h = 0;
    PF_CUDA(cudaMemcpy(&h, status, 4, cudaMemcpyDeviceToHost), err);
    if (h) {
      err = "Philox stream: draw window too small (internal error)";
      return PF_ECUDA;
    }
    return PF_OK;
  }
};

// One kernel launch as issued by the launch helpers: the per-frame step
// graph (run_enqueue, F == 1) re-issues a step by updating its kernel nodes
// with the recorded arguments instead of launching.
struct LaunchRec {
  const void* fn;
  dim3 grid, block;
  size_t smem;
  std::vector<unsigned char> args;
};

// host frames are uploaded in this many chunks on a copy stream; each
// chunk's likelihood maps start as soon as it lands (pf_run)
constexpr int kUploadChunks = 8;
// host frames up to this size are staged through a pinned buffer by the
// synchronous calls (a per-frame step's frame is 16 KB at 128x128)
constexpr size_t kStageBytes = 1u << 20;

struct pf_handle {
  int precision = 0, km = 0;
  long long K = 0;
  int W = 0, H = 0, r = 0, Hm = 0, Wm = 0;
  int n_tracks = 1, n_videos = 1;
  int tpb = 256, vpt = 4;
  pf_params params{};
  int n_off = 0;
  double start_x = 0, start_y = 0;
  int device = 0;
  cudaStream_t stream = nullptr;
  int n_tiles = 0, n_pad = 1, Q = 52, tpb_table = 32, n_chunks = 1;
  unsigned long long* tsync = nullptr;
  long long* tagg = nullptr;
  double* troots = nullptr;
  size_t rs = 8, vs = 16;
  void* X[2] = {nullptr, nullptr};
  void* C[2] = {nullptr, nullptr};
  int cur = 0;
  double* rec_m = nullptr;
  long long *rec_S = nullptr, *rec_X = nullptr, *rec_Y = nullptr;
  long long* tab_s = nullptr;
  double *tab_O = nullptr, *tab_invM = nullptr, *u = nullptr;
  int2* win = nullptr;  // [track][tile] source window for the next frame
  unsigned long long* x0 = nullptr;
  ulonglong2* tj = nullptr;
  ulonglong2* tt = nullptr;
  bool pdl = true;
  unsigned short* exp16 = nullptr;
  int* exp16q = nullptr;  // rint(exp16 * 2^20): the fused FP16 kernel's weights
  void* zig = nullptr;
  int2* d_offs = nullptr;
  short* d_plan = nullptr;
  short2* d_leaves = nullptr;
  int2* d_runs = nullptr;  // pf_map_wide_runs: row-prefix displacements per template run
  int n_runs = 0;
  bool map_runs = false;
  int map_runs_band = 8;
  size_t map_runs_smem = 0;
  int n_plan = 0;
  uint8_t* d_frames = nullptr;
  size_t frames_cap = 0;
  void* d_maps = nullptr;
  size_t maps_cap = 0;
  double* d_traj = nullptr;
  size_t traj_cap = 0;
  int* d_degen = nullptr;
  int* h_degen = nullptr;  // pinned host copy of d_degen
  long long* dbg_anc = nullptr;
  void* dbg_L = nullptr;
  long long frame_counter = 0;
  std::string err;
  cudaEvent_t ev[6] = {};
  cudaStream_t cstream = nullptr;          // host-frame uploads, chunked ahead of the maps
  cudaEvent_t cev[kUploadChunks] = {};     // per-chunk upload done
  float timings[6] = {0};
  bool timings_stale = false;  // timings[] not yet read from the last run's events
  int timings_F = 0;
  int64_t launches = 0;
  int degenerate_frame = -1;
  size_t map_smem = 0, fused_smem = 0, fused_smem_base = 0;
  int map_band = 32;
  bool map_wide_img = false;  // FP32 / FP64 term-image map kernel
  int map_wide_band = 8;
  size_t map_wide_smem = 0;
  bool map_img = false;  // binary16 term-image map kernel
  bool profiling = false;
  std::vector<cudaEvent_t> pev;  // 3 per frame when profiling
  bool use_graphs = true;
  cudaGraphExec_t gexec = nullptr;
  long long g_start = -1;
  int g_cur = -1, g_F = -1;
  const void* g_maps = nullptr;
  const void* g_traj = nullptr;
  const void* g_est = nullptr;  // host-mapped trajectory the run graph's tables write (or null)
  // sharding (pf_shard_*): this handle holds global tiles [tile0, tile0 + nl)
  long long Kl = 0;  // particles per track held here (== K unless sharded)
  int nl = 0;        // tiles per track held here (== n_tiles unless sharded)
  int tile0 = 0, n_shards = 1, shard = 0, shard_tiles = 0, sh_chunks = 0;
  void* peer[PF_MAX_SHARDS][8] = {};  // per shard: X0, X1, C0, C1, tab_s, tab_O, tab_invM, win
  bool peer_ipc[PF_MAX_SHARDS] = {};
  long long *sh_mass = nullptr, *sh_ctot = nullptr, *sh_send = nullptr, *sh_gsum = nullptr;
  double* sh_croots = nullptr;
  unsigned long long* sh_gmax = nullptr;
  cudaEvent_t xev = nullptr;
  int sh_F = 0;
  // unsharded track too large for the co-resident chunked table: run the
  // sharded table kernels with one shard (no spinning across CTAs)
  bool split_table = false;
  unsigned long long* d_trace = nullptr;  // pf_set_trace: [frame][n_tiles + n_chunks][8]
  size_t trace_cap = 0;
  bool tracing = false;
  // stream-ordered calls (pf_run_async): caller-stream handoff events, and
  // whether a run is enqueued but not yet completed (pf_sync)
  cudaEvent_t xin = nullptr, xout = nullptr;
  bool pending = false;
  int pending_F = 0;
  // pf_set_state: the next frame runs with identity ancestors (injected state)
  bool ident_next = false;
  bool g_ident = false;
  // rng = numpy-philox (pf_set_rng_philox): every frame's 2K normals and
  // uniform come from the reference's own stream, generated before the frames
  bool philox = false;
  PhxGen phx;
  // the next fused launch follows a kernel whose results it reads without a
  // grid dependency wait (likelihood maps, Philox draws): launch it without
  // programmatic overlap
  bool serialize_next = false;
  // per-frame step graph (F == 1): [frame H2D] -> maps [-> Philox draws] ->
  // fused -> table, re-launched with updated kernel-node arguments
  std::vector<LaunchRec>* rec = nullptr;  // launch helpers append here
  bool rec_only = false;                  // ... and do not launch
  cudaGraph_t sg = nullptr;
  cudaGraphExec_t sgx = nullptr;
  cudaGraphNode_t sg_node[3] = {};  // maps, fused, table
  int sg_on_dev = -1;
  const void *sg_frames = nullptr, *sg_maps = nullptr, *sg_traj = nullptr, *sg_noise = nullptr;
  bool sg_ident = false;
  // pinned staging of the synchronous calls (pf_run / pf_step)
  uint8_t* h_stage = nullptr;
  double* h_traj = nullptr;
  size_t h_traj_cap = 0;
  double* traj_user = nullptr;
  size_t traj_bytes = 0;
  // one-frame synchronous steps: the tile table writes the estimate and the
  // degeneracy flag straight into host-mapped memory (no copy back)
  double* h_est_map = nullptr;  // [track][frame][2] trajectory of the run
  size_t est_map_cap = 0;       // bytes
  int* h_deg_map = nullptr;     // [track] first degenerate frame of the run (INT_MAX = none)
  double* d_est_map = nullptr;
  int* d_deg_map = nullptr;
  bool zc_step = false;     // the run being launched writes its results to the mapped buffers
  bool zc_pending = false;  // the enqueued run's result is in the mapped buffers
  double* noise_all = nullptr;  // [F][K][2]
  size_t noise_cap = 0;
  double* u_all = nullptr;  // [F]
  size_t u_cap = 0;
  const void* g_noise = nullptr;
};

// the fused kernel's instantiations live in their own translation units
// (pf_fused_sel.cuh, built in parallel); these select among them
typedef pf_fused_fn fused_fn;
template <int M, bool PK = true, bool DBG = false>
static fused_fn fused_for_tpb(int tpb) {
  return pf_fused_sel(M, PK, DBG, tpb);
}
template <int M>
static fused_fn fused_sharded(int tpb) {
  return pf_fused_sel_sharded(M, tpb);
}
template <int M, bool PK>
static fused_fn fused_nz(int tpb) {
  return pf_fused_sel_nz(M, PK, tpb);
}
// dbg: the instantiation with the trace / debug-capture hooks (pf_set_trace,
// pf_get_debug); the production kernels carry neither
template <bool DBG>
static fused_fn fused_unsharded(const pf_handle* h) {
  if (h->km == 2 && h->precision == PF_FP16) return fused_for_tpb<2, false, DBG>(h->tpb);  // scalar lanes
  return h->km == 0 ? fused_for_tpb<0, true, DBG>(h->tpb)
                    : h->km == 1 ? fused_for_tpb<1, true, DBG>(h->tpb) : fused_for_tpb<2, true, DBG>(h->tpb);
}
static bool fused_dbg(const pf_handle* h) { return h->n_shards == 1 && (h->dbg_anc != nullptr || h->tracing); }
static fused_fn fused_kernel(const pf_handle* h, int dbg = -1) {
  if (h->n_shards > 1)
    return h->km == 0 ? fused_sharded<0>(h->tpb) : h->km == 1 ? fused_sharded<1>(h->tpb) : fused_sharded<2>(h->tpb);
  if (h->philox) {
    if (h->km == 2) return h->precision == PF_FP16 ? fused_nz<2, false>(h->tpb) : fused_nz<2, true>(h->tpb);
    return h->km == 0 ? fused_nz<0, true>(h->tpb) : fused_nz<1, true>(h->tpb);
  }
  const bool d = dbg < 0 ? fused_dbg(h) : dbg != 0;
  return d ? fused_unsharded<true>(h) : fused_unsharded<false>(h);
}
// Dynamic shared memory of the fused launches.  When a frame's whole grid is
// one wave (C1 / C2 sizes), the footprint is padded so that no SM holds more
// than ceil(CTAs / SMs) of them: the block scheduler otherwise packs up to the
// occupancy limit on some SMs (e.g. 10 FP16 CTAs where 6.6 is the mean), and
// the frame waits for the most loaded SM (C2 FP16 +7%, same-box A/B).
static cudaError_t set_fused_smem(pf_handle* h) {
  h->fused_smem = h->fused_smem_base;
  int cap = 0;
  if (const char* mb = std::getenv("PF_FUSED_MAXB")) cap = std::atoi(mb);  // A/B knob (0: no padding)
  int per_sm = 0, sms = 0, sm_smem = 0, resv = 0;
  const void* k0 = (const void*)fused_kernel(h, 0);
  cudaError_t e = cudaFuncSetAttribute(k0, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h->fused_smem);
  if (e == cudaSuccess && h->n_shards == 1 && (cap > 0 || std::getenv("PF_FUSED_MAXB") == nullptr) &&
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device) == cudaSuccess &&
      cudaDeviceGetAttribute(&sm_smem, cudaDevAttrMaxSharedMemoryPerMultiprocessor, h->device) == cudaSuccess &&
      cudaDeviceGetAttribute(&resv, cudaDevAttrReservedSharedMemoryPerBlock, h->device) == cudaSuccess &&
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k0, h->tpb, h->fused_smem) == cudaSuccess) {
    const long long total = (long long)h->nl * h->n_tracks;
    if (cap <= 0 && total <= (long long)per_sm * sms) cap = (int)((total + sms - 1) / sms);
    if (cap > 0 && cap < per_sm) h->fused_smem = std::max(h->fused_smem, (size_t)(sm_smem / (cap + 1) - resv + 16));
  }
  cudaGetLastError();
  e = cudaFuncSetAttribute(k0, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h->fused_smem);
  if (e == cudaSuccess && h->n_shards == 1 && !h->philox)
    e = cudaFuncSetAttribute((const void*)fused_kernel(h, 1), cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)h->fused_smem);
  return e;
}

// launch with programmatic stream serialization (PDL): the kernel may begin
// before its predecessor finishes and waits (griddepcontrol.wait) where it
// consumes the predecessor's results
template <typename Args>
static cudaError_t launch_pdl(const pf_handle* h, const void* fn, dim3 grid, dim3 block, size_t smem, Args args,
                              bool allow = true) {
  if (h->rec) {
    LaunchRec r{fn, grid, block, smem, std::vector<unsigned char>(sizeof(Args))};
    std::memcpy(r.args.data(), &args, sizeof(Args));
    h->rec->push_back(std::move(r));
    if (h->rec_only) return cudaSuccess;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = h->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = (h->pdl && allow) ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  void* params[1] = {&args};
  return cudaLaunchKernelExC(&cfg, fn, params);
}

static int grow(void** p, size_t* cap, size_t bytes, std::string& err) {
  if (*cap >= bytes) return PF_OK;
  if (*p) cudaFree(*p);
  *p = nullptr;
  *cap = 0;
  PF_CUDA(cudaMalloc(p, bytes), err);
  *cap = bytes;
  return PF_OK;
}

extern "C" {

const char* pf_version(void) { return "pf_b200 0.1 (sm_100a)"; }
const char* pf_global_error(void) { return g_err.c_str(); }
const char* pf_last_error(const pf_handle* h) { return h ? h->err.c_str() : g_err.c_str(); }

int pf_exp16_table(uint16_t* out) {
  if (!out) return PF_EINVAL;
  build_exp16(out);
  return PF_OK;
}

int pf_exp16_device(uint16_t* out, int32_t device) {
  if (!out) return PF_EINVAL;
  PF_CUDA(cudaSetDevice(device), g_err);
  std::vector<uint16_t> host(65536);
  build_exp16(host.data());
  unsigned short *tab = nullptr, *res = nullptr;
  PF_CUDA(cudaMalloc(&tab, 65536 * 2), g_err);
  PF_CUDA(cudaMalloc(&res, 65536 * 2), g_err);
  PF_CUDA(cudaMemcpy(tab, host.data(), 65536 * 2, cudaMemcpyHostToDevice), g_err);
  pfk::pf_exp16_fast_check<<<256, 256>>>(tab, res);
  PF_CUDA(cudaGetLastError(), g_err);
  PF_CUDA(cudaMemcpy(out, res, 65536 * 2, cudaMemcpyDeviceToHost), g_err);
  cudaFree(tab);
  cudaFree(res);
  return PF_OK;
}

int pf_destroy(pf_handle* h) {
  if (!h) return PF_OK;
  cudaSetDevice(h->device);
  void* ptrs[] = {h->X[0], h->X[1], h->C[0], h->C[1], h->rec_m, h->rec_S, h->rec_X, h->rec_Y, h->tab_s, h->tab_O,
                  h->tab_invM, h->win, h->u, h->x0, h->tj, h->tt, h->tsync, h->tagg, h->troots, h->exp16, h->exp16q, h->zig, h->d_offs, h->d_plan, h->d_leaves, h->d_runs, h->d_frames,
                  h->d_maps, h->d_traj, h->d_degen, h->dbg_anc, h->dbg_L, h->d_trace};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  void* sptrs[] = {h->sh_mass, h->sh_ctot, h->sh_croots, h->sh_send, h->sh_gsum, h->sh_gmax};
  for (void* p : sptrs)
    if (p) cudaFree(p);
  for (int sh = 0; sh < PF_MAX_SHARDS; ++sh)
    if (h->peer_ipc[sh])
      for (int i = 0; i < 8; ++i)
        if (h->peer[sh][i]) cudaIpcCloseMemHandle(h->peer[sh][i]);
  if (h->pending) cudaStreamSynchronize(h->stream);
  if (h->sgx) cudaGraphExecDestroy(h->sgx);
  if (h->sg) cudaGraphDestroy(h->sg);
  h->phx.release();
  if (h->h_stage) cudaFreeHost(h->h_stage);
  if (h->h_traj) cudaFreeHost(h->h_traj);
  if (h->h_est_map) cudaFreeHost(h->h_est_map);
  if (h->h_deg_map) cudaFreeHost(h->h_deg_map);
  if (h->noise_all) cudaFree(h->noise_all);
  if (h->u_all) cudaFree(h->u_all);
  if (h->xev) cudaEventDestroy(h->xev);
  if (h->xin) cudaEventDestroy(h->xin);
  if (h->xout) cudaEventDestroy(h->xout);
  if (h->h_degen) cudaFreeHost(h->h_degen);
  for (auto& e : h->ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : h->pev) cudaEventDestroy(e);
  for (auto& e : h->cev)
    if (e) cudaEventDestroy(e);
  if (h->cstream) cudaStreamDestroy(h->cstream);
  if (h->gexec) cudaGraphExecDestroy(h->gexec);
  if (h->stream) cudaStreamDestroy(h->stream);
  delete h;
  return PF_OK;
}

static int validate(const pf_config* c, std::string& err) {
  if (!c) {
    err = "null config";
    return PF_EINVAL;
  }
  if (c->precision < PF_FP64 || c->precision > PF_FP16_PACKED) {
    err = "unknown precision";
    return PF_EINVAL;
  }
  if (c->K < 2) {
    err = "particle count must be at least 2";
    return PF_EINVAL;
  }
  if (c->K > (1LL << 31) - 1) {
    err = "particle count exceeds the 2^31-1 per-track bound";
    return PF_EINVAL;
  }
  if (c->precision == PF_FP16_PACKED && (c->K % 2)) {
    err = "packed binary16 mode requires an even particle count";
    return PF_EINVAL;
  }
  if (c->width < 1 || c->height < 1 || c->n_tracks < 1 || c->n_videos < 1 || c->n_offsets < 1 ||
      c->n_offsets > 4096 || !c->offsets_xy || !c->seeds) {
    err = "bad shape / template / seeds";
    return PF_EINVAL;
  }
  int tpb = c->tpb ? c->tpb : 128;
  if (tpb != 32 && tpb != 64 && tpb != 128 && tpb != 256 && tpb != 512 && tpb != 1024) {
    err = "tpb must be a power of two in [32, 1024]";
    return PF_EINVAL;
  }
  return PF_OK;
}

static int create_impl(pf_handle** out, const pf_config* cfg, int n_shards, int shard) {
  if (!out) return PF_EINVAL;
  *out = nullptr;
  int rc = validate(cfg, g_err);
  if (rc) return rc;
  if (n_shards < 1 || n_shards > PF_MAX_SHARDS || shard < 0 || shard >= n_shards ||
      (n_shards > 1 && cfg->n_tracks != 1)) {
    g_err = "bad shard layout (1..8 shards of one track)";
    return PF_EINVAL;
  }
  pf_handle* h = new pf_handle();
  h->precision = cfg->precision;
  h->km = kmode_of(cfg->precision);
  h->K = cfg->K;
  h->W = cfg->width;
  h->H = cfg->height;
  h->n_tracks = cfg->n_tracks;
  h->n_videos = cfg->n_videos;
  // default threads per block per precision (measured, bench TPB sweeps):
  // FP16 / FP32 prefer 128 threads while the grid fits in about one wave
  // (C2: FP32 3.9e10 at 128 vs 3.3e10 at 256), 256 beyond; FP64 256
  {
    const long long ctas = ((cfg->K + PF_TILE - 1) / PF_TILE) * (long long)cfg->n_tracks;
    h->tpb = cfg->tpb ? cfg->tpb : (cfg->precision != PF_FP64 && ctas <= 2048 ? 128 : 256);
  }
  if (n_shards > 1 && h->tpb != 128) h->tpb = 256;  // sharded kernels exist for 128 / 256 threads
  h->vpt = h->tpb >= 1024 ? 1 : h->tpb >= 512 ? 2 : h->tpb >= 256 ? 4 : 8;
  h->params = cfg->params;
  h->n_off = cfg->n_offsets;
  h->start_x = cfg->start_x;
  h->start_y = cfg->start_y;
  h->device = cfg->device;
  int r = 0;
  for (int i = 0; i < cfg->n_offsets; ++i)
    r = std::max(r, std::max(std::abs(cfg->offsets_xy[2 * i]), std::abs(cfg->offsets_xy[2 * i + 1])));
  h->r = r;
  h->Hm = h->H + 2 * r;
  h->Wm = h->W + 2 * r;
  h->rs = real_size(h->km);
  h->vs = 2 * h->rs;
  h->n_tiles = (int)((h->K + PF_TILE - 1) / PF_TILE);
  h->n_shards = n_shards;
  h->shard = shard;
  if (n_shards > 1) {
    // power-of-two tiles per shard: every shard's estimate subtree is a node
    // of the single-GPU canonical tree (bit-identical results)
    h->shard_tiles = next_pow2((h->n_tiles + n_shards - 1) / n_shards);
    if ((long long)(n_shards - 1) * h->shard_tiles >= h->n_tiles) {
      g_err = "too few tiles for this many shards (every shard must hold particles)";
      delete h;
      return PF_EINVAL;
    }
    h->tile0 = shard * h->shard_tiles;
    h->nl = std::min(h->n_tiles - h->tile0, h->shard_tiles);
    h->Kl = std::min(h->K, (long long)(h->tile0 + h->nl) * PF_TILE) - (long long)h->tile0 * PF_TILE;
    h->sh_chunks = (h->nl + pfk::kShardChunk - 1) / pfk::kShardChunk;
  } else {
    h->shard_tiles = h->n_tiles;
    h->nl = h->n_tiles;
    h->Kl = h->K;
  }
  h->n_pad = next_pow2(h->n_tiles);
  int lg = 0;
  while ((1LL << lg) < h->n_tiles) ++lg;
  h->Q = 52 - lg;
  // tile table: one tile per thread; a single CTA up to 1024 tiles (the
  // cross-CTA exchanges cost more than they save there), chunks of 256 above
  h->tpb_table = h->n_pad <= 1024 ? std::max(32, h->n_pad) : 256;
  if (const char* tt = std::getenv("PF_TABLE_TPB")) {  // A/B knob: tiles per table CTA
    const int v = std::atoi(tt);
    if (v >= 32 && v <= 1024 && (v & (v - 1)) == 0) h->tpb_table = std::min(h->tpb_table, v);
  }
  h->n_chunks = (h->n_tiles + h->tpb_table - 1) / h->tpb_table;
  std::string& e = h->err;
#define CK(x)                    \
  do {                           \
    int _r = (x);                \
    if (_r) {                    \
      g_err = h->err;            \
      pf_destroy(h);             \
      return _r;                 \
    }                            \
  } while (0)
  auto cudack = [&](cudaError_t ce, const char* what) -> int {
    if (ce != cudaSuccess) {
      e = std::string("CUDA error ") + cudaGetErrorString(ce) + " at " + what;
      return PF_ECUDA;
    }
    return PF_OK;
  };
  CK(cudack(cudaSetDevice(h->device), "cudaSetDevice"));
  CK(init_device_tables(h->device, e));
  CK(cudack(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking), "stream"));
  for (auto& ev : h->ev) CK(cudack(cudaEventCreate(&ev), "event"));
  const size_t KT = (size_t)h->Kl * h->n_tracks;
  const size_t NT = (size_t)h->nl * h->n_tracks;
  for (int i = 0; i < 2; ++i) {
    CK(cudack(cudaMalloc(&h->X[i], KT * h->vs), "X"));
    // slack: 16-byte rounded bulk copies, and the search's 4-entry probe (up
    // to three entries read past a track's last local CDF value)
    CK(cudack(cudaMalloc(&h->C[i], KT * h->rs + 32), "C"));
  }
  CK(cudack(cudaMalloc(&h->rec_m, NT * 8), "rec"));
  CK(cudack(cudaMalloc(&h->rec_S, NT * 8), "rec"));
  CK(cudack(cudaMalloc(&h->rec_X, NT * 8), "rec"));
  CK(cudack(cudaMalloc(&h->rec_Y, NT * 8), "rec"));
  CK(cudack(cudaMalloc(&h->tab_s, NT * 8), "tab"));
  CK(cudack(cudaMalloc(&h->tab_O, NT * 8), "tab"));
  CK(cudack(cudaMalloc(&h->tab_invM, NT * 8), "tab"));
  CK(cudack(cudaMalloc(&h->win, NT * sizeof(int2)), "win"));
  CK(cudack(cudaMalloc(&h->u, h->n_tracks * 8), "u"));
  CK(cudack(cudaMalloc(&h->d_degen, h->n_tracks * sizeof(int)), "degen"));
  CK(cudack(cudaMalloc(&h->tsync, (size_t)h->n_tracks * 4 * 8), "tsync"));
  CK(cudack(cudaMemset(h->tsync, 0, (size_t)h->n_tracks * 4 * 8), "tsync"));
  CK(cudack(cudaMalloc(&h->tagg, (size_t)h->n_tracks * h->n_chunks * 8), "tagg"));
  CK(cudack(cudaMalloc(&h->troots, (size_t)h->n_tracks * h->n_chunks * 3 * 8), "troots"));
  // per-track LCG seed states
  std::vector<unsigned long long> x0(h->n_tracks);
  for (int i = 0; i < h->n_tracks; ++i) x0[i] = pfr::seed_state(cfg->seeds[i]);
  CK(cudack(cudaMalloc(&h->x0, h->n_tracks * 8), "x0"));
  CK(cudack(cudaMemcpy(h->x0, x0.data(), h->n_tracks * 8, cudaMemcpyHostToDevice), "x0"));
  // per-virtual-thread jumps f^(2 v VPT)
  const int nv = PF_TILE / h->vpt;
  std::vector<ulonglong2> tj(nv);
  for (int v = 0; v < nv; ++v) {
    pfr::Affine f = pfr::affine_pow(2ULL * v * h->vpt);
    tj[v] = make_ulonglong2(f.a, f.c);
  }
  CK(cudack(cudaMalloc(&h->tj, nv * sizeof(ulonglong2)), "tj"));
  CK(cudack(cudaMemcpy(h->tj, tj.data(), nv * sizeof(ulonglong2), cudaMemcpyHostToDevice), "tj"));
  // per-tile jumps f^(2 * tile * PF_TILE) and f^(2K)
  {
    std::vector<ulonglong2> tt(h->nl);  // local tile b is global tile tile0 + b
    const pfr::Affine step = pfr::affine_pow(2ULL * PF_TILE);
    pfr::Affine f = pfr::affine_pow(2ULL * PF_TILE * (unsigned long long)h->tile0);
    for (int b = 0; b < h->nl; ++b) {
      tt[b] = make_ulonglong2(f.a, f.c);
      f = pfr::compose(step, f);
    }
    CK(cudack(cudaMalloc(&h->tt, h->nl * sizeof(ulonglong2)), "tt"));
    CK(cudack(cudaMemcpy(h->tt, tt.data(), h->nl * sizeof(ulonglong2), cudaMemcpyHostToDevice), "tt"));
  }
  // exp16 table
  std::vector<uint16_t> ex(65536);
  build_exp16(ex.data());
  CK(cudack(cudaMalloc(&h->exp16, 65536 * 2), "exp16"));
  CK(cudack(cudaMemcpy(h->exp16, ex.data(), 65536 * 2, cudaMemcpyHostToDevice), "exp16"));
  {  // the same weights as weight_q<M_FP16>: rint(f32(w) * 2^20), round half to even
    std::vector<int> exq(65536);
    for (int i = 0; i < 65536; ++i) {
      const double v = std::nearbyint(f16_to_f64(ex[i]) * 1048576.0);
      exq[i] = std::isfinite(v) && v < 2147483647.0 ? (int)v : INT_MAX;
    }
    CK(cudack(cudaMalloc(&h->exp16q, 65536 * 4), "exp16q"));
    CK(cudack(cudaMemcpy(h->exp16q, exq.data(), 65536 * 4, cudaMemcpyHostToDevice), "exp16q"));
  }
  // ziggurat fast-path tables, packed for 16-byte smem staging: 256 x (ki >> 20)
  // then 256 x wi; binary16 modes: 256 x {ki >> 29, f32(wi * 2^29)} (the
  // binary32 fast path on the word's high 32 bits, oracle/rng.py)
  {
    std::vector<unsigned char> zt(pfk::kZigBytes, 0);
    for (int i = 0; i < 256; ++i) {
      if (h->km == 2) {
        double wi;
        std::memcpy(&wi, &PF_ZIG_WI_BITS_HOST[i], 8);
        const uint32_t k32 = (uint32_t)(PF_ZIG_KI_HOST[i] >> 29);
        const float w32 = (float)std::ldexp(wi, 29);  // exact scaling, one RN to binary32
        std::memcpy(zt.data() + 8 * i, &k32, 4);
        std::memcpy(zt.data() + 8 * i + 4, &w32, 4);
        continue;
      }
      uint32_t khi = (uint32_t)(PF_ZIG_KI_HOST[i] >> 20);
      std::memcpy(zt.data() + 4 * i, &khi, 4);
      std::memcpy(zt.data() + 1024 + 8 * i, &PF_ZIG_WI_BITS_HOST[i], 8);
    }
    CK(cudack(cudaMalloc(&h->zig, pfk::kZigBytes), "zig"));
    CK(cudack(cudaMemcpy(h->zig, zt.data(), pfk::kZigBytes, cudaMemcpyHostToDevice), "zig"));
  }
  // template + pairwise plan
  std::vector<int2> offs(h->n_off);
  for (int i = 0; i < h->n_off; ++i) offs[i] = make_int2(cfg->offsets_xy[2 * i], cfg->offsets_xy[2 * i + 1]);
  CK(cudack(cudaMalloc(&h->d_offs, h->n_off * sizeof(int2)), "offs"));
  CK(cudack(cudaMemcpy(h->d_offs, offs.data(), h->n_off * sizeof(int2), cudaMemcpyHostToDevice), "offs"));
  std::vector<long long> ls;
  std::vector<int> ll, ops;
  pw_plan(0, h->n_off, ls, ll, ops);
  h->n_plan = (int)ops.size();
  std::vector<short> plan(ops.begin(), ops.end());
  std::vector<short2> leaves(h->n_plan, make_short2(0, 0));
  for (size_t i = 0; i < ls.size(); ++i) leaves[i] = make_short2((short)ls[i], (short)ll[i]);
  CK(cudack(cudaMalloc(&h->d_plan, h->n_plan * sizeof(short)), "plan"));
  CK(cudack(cudaMalloc(&h->d_leaves, h->n_plan * sizeof(short2)), "plan"));
  CK(cudack(cudaMemcpy(h->d_plan, plan.data(), h->n_plan * sizeof(short), cudaMemcpyHostToDevice), "plan"));
  CK(cudack(cudaMemcpy(h->d_leaves, leaves.data(), h->n_plan * sizeof(short2), cudaMemcpyHostToDevice), "plan"));
  // launch geometry
  h->map_band = h->W >= 512 ? 8 : 32;
  size_t rows_bytes = (size_t)(h->map_band + 2 * h->r) * h->W + 32;
  h->map_smem = 16 + 256 * h->rs + h->n_off * sizeof(int2) + h->n_plan * (sizeof(short) + sizeof(short2)) + 16 +
                rows_bytes;
  h->fused_smem_base = h->km == 0 ? pfk::fused_smem_bytes<0>() : h->km == 1 ? pfk::fused_smem_bytes<1>()
                                                                           : pfk::fused_smem_bytes<2>();
  CK(cudack(set_fused_smem(h), "fused smem attr"));
  // binary16: the term-image kernel when its shared memory fits
  h->map_img = false;
  if (h->km == 2) {
    const pfk::MapHalfGeom g = pfk::map_half_geom(h->W, h->H, h->r, h->n_off);
    if (g.smem <= 200 * 1024) {
      h->map_img = true;
      CK(cudack(cudaFuncSetAttribute(pfk::pf_map_half_img<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)g.smem),
                "map smem attr"));
      CK(cudack(cudaFuncSetAttribute(pfk::pf_map_half_img<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)g.smem),
                "map smem attr"));
    }
  }
  // FP32 / FP64: the term-image kernel for single-leaf templates when a band fits
  h->map_wide_img = false;
  if (h->km != 2 && h->n_plan == 1) {
    int band = h->W >= 512 ? 8 : 32;
    while (band > 1 && pfk::map_wide_geom(h->W, h->r, h->n_off, h->rs, band).smem > 200 * 1024) band /= 2;
    const pfk::MapWideGeom g = pfk::map_wide_geom(h->W, h->r, h->n_off, h->rs, band);
    if (g.smem <= 200 * 1024 && std::getenv("PF_MAP_GENERIC") == nullptr) {
      h->map_wide_img = true;
      h->map_wide_band = band;
      h->map_wide_smem = g.smem;
      CK(cudack(cudaFuncSetAttribute(h->km == 0 ? (const void*)pfk::pf_map_wide_img<double>
                                                : (const void*)pfk::pf_map_wide_img<float>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g.smem),
                "map smem attr"));
    }
  }
  // FP32 / FP64 with integral means and a small enough template: every term
  // and partial sum is an exact integer, so the map comes from integer row
  // prefix sums over the template's horizontal runs (pf_map_wide_runs)
  if (h->km != 2 && std::getenv("PF_MAP_GENERIC") == nullptr) {
    const double bg = h->params.bg_mean, fg = h->params.fg_mean;
    bool ok = bg == std::floor(bg) && fg == std::floor(fg) && std::fabs(bg) <= 1024 && std::fabs(fg) <= 1024;
    long long T = 0;
    if (ok)
      for (int v = 0; v < 256; ++v) {
        const long long ib = (long long)bg, ifg = (long long)fg;
        T = std::max(T, std::llabs((v - ib) * (v - ib) - (v - ifg) * (v - ifg)));
      }
    ok = ok && (long long)h->n_off * T < (1LL << 24);
    std::vector<std::pair<int, int>> so(h->n_off);
    for (int i = 0; i < h->n_off; ++i) so[i] = {cfg->offsets_xy[2 * i + 1], cfg->offsets_xy[2 * i]};  // (dy, dx)
    std::sort(so.begin(), so.end());
    for (int i = 1; i < h->n_off && ok; ++i) ok = so[i] != so[i - 1];  // a multiset is not a union of runs
    const int Wz = h->W + 4 * h->r + 1;
    ok = ok && (long long)Wz * T < (1LL << 31);
    if (ok) {
      std::vector<int2> runs;
      for (int i = 0; i < h->n_off;) {
        int j = i;
        while (j + 1 < h->n_off && so[j + 1].first == so[i].first && so[j + 1].second == so[j].second + 1) ++j;
        const int dy = so[i].first, dx0 = so[i].second, dx1 = so[j].second;
        runs.push_back(make_int2((dy + h->r) * Wz + h->r + dx1 + 1, (dy + h->r) * Wz + h->r + dx0));
        i = j + 1;
      }
      int band = h->W >= 512 ? 8 : 32;
      while (band > 1 && pfk::map_runs_geom(h->W, h->r, (int)runs.size(), band).smem > 200 * 1024) band /= 2;
      const pfk::MapRunsGeom g = pfk::map_runs_geom(h->W, h->r, (int)runs.size(), band);
      if (g.smem <= 200 * 1024) {
        h->n_runs = (int)runs.size();
        CK(cudack(cudaMalloc(&h->d_runs, runs.size() * sizeof(int2)), "runs"));
        CK(cudack(cudaMemcpy(h->d_runs, runs.data(), runs.size() * sizeof(int2), cudaMemcpyHostToDevice), "runs"));
        h->map_runs = true;
        h->map_runs_band = band;
        h->map_runs_smem = g.smem;
        CK(cudack(cudaFuncSetAttribute(h->km == 0 ? (const void*)pfk::pf_map_wide_runs<double>
                                                  : (const void*)pfk::pf_map_wide_runs<float>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g.smem),
                  "map smem attr"));
      }
    }
  }
  if (h->map_smem > 48 * 1024) {
    cudaError_t ce = cudaSuccess;
    if (h->km == 0)
      ce = cudaFuncSetAttribute(pfk::pf_map_wide<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h->map_smem);
    else if (h->km == 1)
      ce = cudaFuncSetAttribute(pfk::pf_map_wide<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h->map_smem);
    else
      ce = cudaFuncSetAttribute(pfk::pf_map_half, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h->map_smem);
    CK(cudack(ce, "map smem attr"));
  }
  if (n_shards == 1) {
    // the chunked table exchanges through spinning CTAs: all of a frame's
    // chunks must be co-resident, else the sharded kernels run it (1 shard)
    int per_sm = 0, sms = 0;
    const void* tk = h->km == 0 ? (const void*)pfk::pf_tile_table<0>
                     : h->km == 1 ? (const void*)pfk::pf_tile_table<1> : (const void*)pfk::pf_tile_table<2>;
    CK(cudack(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tk, h->tpb_table, 0), "occupancy"));
    CK(cudack(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device), "attr"));
    const char* force = std::getenv("PF_FORCE_SPLIT_TABLE");  // test knob: exercise the split path small
    // (one track's chunks wait only for each other and are launched
    // contiguously, so the bound is per track; single-chunk tables never spin)
    if ((h->n_chunks > 1 && (long long)h->n_chunks > (long long)per_sm * sms / 2) ||
        (force && force[0] == '1' && h->n_tracks == 1)) {
      if (h->n_tracks != 1) {
        e = "too many table chunks for co-residency with several tracks (split the batch)";
        g_err = e;
        pf_destroy(h);
        return PF_EINVAL;
      }
      h->split_table = true;
      h->sh_chunks = (h->nl + pfk::kShardChunk - 1) / pfk::kShardChunk;
    }
  }
  if (n_shards > 1 || h->split_table) {
    CK(cudack(cudaMalloc(&h->sh_mass, (size_t)h->nl * 8), "shard"));
    CK(cudack(cudaMalloc(&h->sh_ctot, (size_t)h->sh_chunks * 8), "shard"));
    CK(cudack(cudaMalloc(&h->sh_croots, (size_t)h->sh_chunks * 3 * 8), "shard"));
    CK(cudack(cudaMalloc(&h->sh_send, 4 * 8), "shard"));
    CK(cudack(cudaMalloc(&h->sh_gsum, (size_t)n_shards * 4 * 8), "shard"));
    CK(cudack(cudaMalloc(&h->sh_gmax, (size_t)n_shards * 8), "shard"));
    if (n_shards > 1) CK(cudack(cudaEventCreateWithFlags(&h->xev, cudaEventDisableTiming), "event"));
  }
  // own buffers as shard `shard`'s source pointers (peers are set later)
  void* own[8] = {h->X[0], h->X[1], h->C[0], h->C[1], h->tab_s, h->tab_O, h->tab_invM, h->win};
  for (int i = 0; i < 8; ++i) h->peer[shard][i] = own[i];
  CK(pf_reset(h, cfg->start_x, cfg->start_y));
#undef CK
  *out = h;
  return PF_OK;
}

int pf_create(pf_handle** out, const pf_config* cfg) { return create_impl(out, cfg, 1, 0); }

int pf_reset(pf_handle* h, double x0, double y0) {
  if (!h) return PF_EINVAL;
  PF_CUDA(cudaSetDevice(h->device), h->err);
  h->start_x = x0;
  h->start_y = y0;
  h->cur = 0;
  h->frame_counter = 0;
  h->ident_next = false;
  h->degenerate_frame = -1;
  const long long n = h->Kl * h->n_tracks;
  const int tb = 256;
  const unsigned nb = (unsigned)((n + tb - 1) / tb);
  if (h->km == 0)
    pfs::fill_start<0><<<nb, tb, 0, h->stream>>>(n, h->X[0], x0, y0);
  else if (h->km == 1)
    pfs::fill_start<1><<<nb, tb, 0, h->stream>>>(n, h->X[0], x0, y0);
  else
    pfs::fill_start<2><<<nb, tb, 0, h->stream>>>(n, h->X[0], x0, y0);
  PF_CUDA(cudaGetLastError(), h->err);
  std::vector<int> dg(h->n_tracks, INT_MAX);
  PF_CUDA(cudaMemcpyAsync(h->d_degen, dg.data(), h->n_tracks * sizeof(int), cudaMemcpyHostToDevice, h->stream),
          h->err);
  PF_CUDA(cudaMemsetAsync(h->tsync, 0, (size_t)h->n_tracks * 4 * 8, h->stream), h->err);
  if (h->philox) {  // the reference stream restarts from its seeded state
    const int rc = h->phx.rewind(h->stream, h->err);
    if (rc) return rc;
  }
  PF_CUDA(cudaStreamSynchronize(h->stream), h->err);
  return PF_OK;
}

// maps of frames [f0, f0 + nf) of a one-video buffer of F frames (nf < 0: all)
static int launch_maps(pf_handle* h, const uint8_t* dframes, int F, int f0 = 0, int nf = -1) {
  if (nf < 0) nf = F;
  if (h->n_videos != 1 && (f0 != 0 || nf != F)) return PF_EINVAL;
  pfk::MapArgs a{};
  a.frames = dframes + (size_t)f0 * h->H * h->W;
  a.n_frames = nf;
  a.H = h->H;
  a.W = h->W;
  a.r = h->r;
  a.Hm = h->Hm;
  a.Wm = h->Wm;
  a.n_off = h->n_off;
  a.offsets = h->d_offs;
  a.plan = h->d_plan;
  a.leaves = h->d_leaves;
  a.n_plan = h->n_plan;
  a.bg = h->params.bg_mean;
  a.fg = h->params.fg_mean;
  a.denom = h->params.likelihood_scale * h->n_off;
  a.bg16 = f64_to_f16(h->params.bg_mean);
  a.fg16 = f64_to_f16(h->params.fg_mean);
  a.s16 = f64_to_f16(1.0 / std::sqrt(h->params.likelihood_scale * h->n_off));
  a.maps = (char*)h->d_maps + (size_t)f0 * h->Hm * h->Wm * h->rs;
  a.band = h->map_band;
  // a handful of frames (per-frame steps): narrow bands, so one frame's map
  // spreads over ~32 CTAs instead of 3-5 long ones (the step's latency)
  const bool few = h->n_videos * nf < 8;
  const int few_band = std::max(1, (h->Hm + 31) / 32);
  dim3 grid((h->Hm + a.band - 1) / a.band, h->n_videos * nf);
  if (h->map_runs) {
    a.band = few ? std::min(h->map_runs_band, few_band) : h->map_runs_band;
    a.runs = h->d_runs;
    a.n_runs = h->n_runs;
    dim3 gw((h->Hm + a.band - 1) / a.band, h->n_videos * nf);
    // C3, 100 frames: 1.2 ms at 512-1024 threads (1.6 at 256) in both modes
    if (h->km == 0)
      PF_CUDA(launch_pdl(h, (const void*)pfk::pf_map_wide_runs<double>, gw, dim3(1024), h->map_runs_smem, a, false), h->err);
    else
      PF_CUDA(launch_pdl(h, (const void*)pfk::pf_map_wide_runs<float>, gw, dim3(1024), h->map_runs_smem, a, false), h->err);
  } else if (h->map_wide_img) {
    a.band = few ? std::min(h->map_wide_band, few_band) : h->map_wide_band;
    dim3 gw((h->Hm + a.band - 1) / a.band, h->n_videos * nf);
    // measured at C3: FP64 3.3 ms per 100 frames at 1024 threads (6.5 at 256,
    // one CTA per SM either way), FP32 2.0 ms at 256 (2.3 at 1024)
    const int mt = h->km == 0 ? 1024 : pfk::kMapWideThreads;
    if (h->km == 0)
      PF_CUDA(launch_pdl(h, (const void*)pfk::pf_map_wide_img<double>, gw, dim3(mt), h->map_wide_smem, a, false), h->err);
    else
      PF_CUDA(launch_pdl(h, (const void*)pfk::pf_map_wide_img<float>, gw, dim3(mt), h->map_wide_smem, a, false), h->err);
  } else if (h->km == 0)
    PF_CUDA(launch_pdl(h, (const void*)pfk::pf_map_wide<double>, grid, dim3(256), h->map_smem, a, false), h->err);
  else if (h->km == 1)
    PF_CUDA(launch_pdl(h, (const void*)pfk::pf_map_wide<float>, grid, dim3(256), h->map_smem, a, false), h->err);
  else if (h->map_img) {
    a.band = few ? few_band : 0;
    const pfk::MapHalfGeom g = pfk::map_half_geom(h->W, h->H, h->r, h->n_off, a.band);
    dim3 gi((h->Hm + g.band - 1) / g.band, h->n_videos * nf);
    if (h->precision == PF_FP16)  // scalar lanes ("fp16")
      PF_CUDA(launch_pdl(h, (const void*)pfk::pf_map_half_img<false>, gi, dim3(pfk::kMapHalfThreads), g.smem, a, false), h->err);
    else
      PF_CUDA(launch_pdl(h, (const void*)pfk::pf_map_half_img<true>, gi, dim3(pfk::kMapHalfThreads), g.smem, a, false), h->err);
  } else
    PF_CUDA(launch_pdl(h, (const void*)pfk::pf_map_half, grid, dim3(256), h->map_smem, a, false), h->err);
  h->launches += 1;
  h->serialize_next = true;
  PF_CUDA(cudaGetLastError(), h->err);
  return PF_OK;
}

static int shard_tables_launch(pf_handle* h, int traj_index, int traj_stride);
static int launch_frame(pf_handle* h, const void* map_slot, long long map_video_stride, int traj_index,
                        int traj_stride);

// one frame: fused kernel + tile table
static int launch_frame(pf_handle* h, const void* map_slot, long long map_video_stride, int traj_index,
                        int traj_stride) {
  if (h->profiling) PF_CUDA(cudaEventRecord(h->pev[3 * traj_index + 0], h->stream), h->err);
  pfk::FusedArgs a{};
  a.K = h->K;
  a.n_tiles = h->n_tiles;
  a.K_local = h->Kl;
  a.n_local = h->nl;
  a.tile0 = h->tile0;
  a.src.n_shards = h->n_shards;
  a.src.shard_tiles = h->shard_tiles;
  for (int sh = 0; sh < h->n_shards; ++sh) {
    a.src.X[sh] = h->peer[sh][h->cur];
    a.src.C[sh] = h->peer[sh][2 + h->cur];
    a.src.ts[sh] = (const long long*)h->peer[sh][4];
    a.src.tO[sh] = (const double*)h->peer[sh][5];
    a.src.tM[sh] = (const double*)h->peer[sh][6];
  }
  a.H = h->H;
  a.W = h->W;
  a.r = h->r;
  a.Wm = h->Wm;
  a.t = (int)h->frame_counter;
  a.ident = (h->frame_counter == 0 || h->ident_next) ? 1 : 0;
  h->ident_next = false;
  a.X_new = h->X[1 - h->cur];
  a.C_new = h->C[1 - h->cur];
  a.u_prev = h->u;
  a.map = map_slot;
  a.map_video_stride = map_video_stride;
  a.n_videos = h->n_videos;
  a.x0 = h->x0;
  a.tj = h->tj;
  a.rec_m = h->rec_m;
  a.rec_S = h->rec_S;
  a.rec_X = h->rec_X;
  a.rec_Y = h->rec_Y;
  a.exp16 = h->exp16;
  a.exp16q = h->exp16q;
  a.drift_x = h->params.drift_x;
  a.drift_y = h->params.drift_y;
  a.std_x = h->params.std_x;
  a.std_y = h->params.std_y;
  a.dbg_anc = h->dbg_anc;
  a.dbg_L = h->dbg_L;
  a.zig = h->zig;
  const pfr::Affine ff = pfr::affine_pow((unsigned long long)h->frame_counter * (2ULL * h->K + 1));
  a.fa = ff.a;
  a.fc = ff.c;
  a.tt = h->tt;
  a.win = h->win;
  a.tmax = h->tsync;
  // sharded / split-table frames are stream-ordered (no PDL, no early release)
  const bool ordered = h->n_shards > 1 || h->split_table;
  a.ready_target = ordered ? 0ULL : (unsigned long long)h->n_chunks * (unsigned long long)h->frame_counter;
  const size_t tr_frame = (size_t)(h->n_tiles + h->n_chunks) * 8;
  a.trace = (h->tracing && h->d_trace) ? h->d_trace + (size_t)traj_index * tr_frame : nullptr;
  a.noise = h->philox ? reinterpret_cast<const double2*>(h->noise_all + (size_t)traj_index * 2 * h->K) : nullptr;
  // a non-identity frame acquires the previous table's release counter instead
  // of waiting on its predecessor grid, so it may overlap only a table kernel:
  // after the maps (or draw) kernels it is launched stream-ordered
  // a one-frame step: launched programmatically behind its map kernel (the
  // draws overlap the map; the map reads wait on the grid dependency --
  // identity frames wait anyway); behind the Philox draw kernels, whose noise
  // the draw phase reads, and in multi-frame runs it stays stream-ordered
  const bool pdl_maps = h->serialize_next && !h->philox && traj_stride == 1 && !ordered;
  a.wait_prev = pdl_maps && !a.ident ? 1 : 0;
  PF_CUDA(launch_pdl(h, (const void*)fused_kernel(h), dim3(h->nl, h->n_tracks), dim3(h->tpb), h->fused_smem, a,
                     !ordered && (!h->serialize_next || pdl_maps)),
          h->err);
  h->serialize_next = false;
  PF_CUDA(cudaGetLastError(), h->err);
  if (h->n_shards > 1) {  // the sharded tables run after the host's collectives (pf_shard_*)
    h->launches += 1;
    return PF_OK;
  }
  if (h->split_table) {  // one shard: the exchanges are the shard's own buffers
    int rc = shard_tables_launch(h, traj_index, traj_stride);
    if (rc) return rc;
    h->launches += 4;
    h->cur = 1 - h->cur;
    h->frame_counter += 1;
    return PF_OK;
  }
  if (h->profiling) PF_CUDA(cudaEventRecord(h->pev[3 * traj_index + 1], h->stream), h->err);
  pfk::TableArgs t{};
  t.K = h->K;
  t.n_tiles = h->n_tiles;
  t.n_pad = h->n_pad;
  t.t = (int)h->frame_counter;
  t.Q = h->Q;
  t.x0 = h->x0;
  t.rec_m = h->rec_m;
  t.rec_S = h->rec_S;
  t.rec_X = h->rec_X;
  t.rec_Y = h->rec_Y;
  t.tab_s = h->tab_s;
  t.tab_O = h->tab_O;
  t.tab_invM = h->tab_invM;
  t.u_out = h->u;
  const pfr::Affine fu =
      pfr::affine_pow((unsigned long long)h->frame_counter * (2ULL * h->K + 1) + 2ULL * (unsigned long long)h->K);
  t.ua = fu.a;
  t.uc = fu.c;
  t.traj = h->d_traj;
  t.traj_stride = traj_stride;
  t.traj_index = traj_index;
  t.degenerate = h->d_degen;
  const void* tk = h->tracing ? (h->km == 0   ? (const void*)pfk::pf_tile_table<0, true>
                                 : h->km == 1 ? (const void*)pfk::pf_tile_table<1, true>
                                              : (const void*)pfk::pf_tile_table<2, true>)
                              : (h->km == 0   ? (const void*)pfk::pf_tile_table<0>
                                 : h->km == 1 ? (const void*)pfk::pf_tile_table<1>
                                              : (const void*)pfk::pf_tile_table<2>);
  t.n_chunks = h->n_chunks;
  t.sync = h->tsync;
  t.agg = h->tagg;
  t.roots = h->troots;
  t.win = h->win;
  t.u_in = h->philox ? h->u_all + traj_index : nullptr;
  t.est_host = h->zc_step ? h->d_est_map : nullptr;  // indexed like traj
  t.deg_host = h->zc_step ? h->d_deg_map : nullptr;
  t.trace = (h->tracing && h->d_trace) ? h->d_trace + (size_t)traj_index * tr_frame + (size_t)h->n_tiles * 8 : nullptr;
  PF_CUDA(launch_pdl(h, tk, dim3(h->n_chunks, h->n_tracks), dim3(h->tpb_table), 0, t), h->err);
  PF_CUDA(cudaGetLastError(), h->err);
  if (h->profiling) PF_CUDA(cudaEventRecord(h->pev[3 * traj_index + 2], h->stream), h->err);
  h->launches += 2;
  h->cur = 1 - h->cur;
  h->frame_counter += 1;
  return PF_OK;
}

// degeneracy flags: copied into pinned host memory on the stream (before the
// run's synchronisation), so the check costs no extra blocking copy
static int queue_degenerate(pf_handle* h) {
  if (!h->h_degen) PF_CUDA(cudaMallocHost(&h->h_degen, (size_t)h->n_tracks * sizeof(int)), h->err);
  PF_CUDA(cudaMemcpyAsync(h->h_degen, h->d_degen, (size_t)h->n_tracks * sizeof(int), cudaMemcpyDeviceToHost,
                          h->stream),
          h->err);
  return PF_OK;
}

static int finish_degenerate(pf_handle* h) {  // after the stream is synchronised
  int m = INT_MAX;
  for (int i = 0; i < h->n_tracks; ++i) m = std::min(m, h->h_degen[i]);
  if (m != INT_MAX) {
    h->degenerate_frame = m;
    h->err = "weight sum degenerated (frame " + std::to_string(m) + ")";
    return PF_EDEGENERATE;
  }
  return PF_OK;
}

// Enqueue a whole-video run on the handle's stream, ordered after `ext`'s
// prior work when ext is given (and `ext` ordered after the run); no host
// synchronisation.  run_complete() waits and reads the timings / degeneracy.
// pageable host memory?  (the synchronous calls stage small copies through
// pinned buffers: a pageable cudaMemcpyAsync is a blocking, driver-staged copy)
static bool is_pageable(const void* p) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return at.type == cudaMemoryTypeUnregistered;
}

// One per-frame step (F == 1) as ONE graph launch: [frame H2D from the pinned
// staging buffer] -> maps [-> Philox draws] -> fused -> table, captured once;
// later steps re-record the three kernels' arguments (frame counter, jump
// constants, buffer parity, frame pointer) without launching and update the
// graph's kernel nodes.  Same kernels, same arguments: same results.
static int step_graph_launch(pf_handle* h, const uint8_t* dframes, int on_device) {
  const size_t map_elems = (size_t)h->Hm * h->Wm;
  const void* frames_key = on_device ? nullptr : (const void*)h->d_frames;
  const bool rebuild = !h->sgx || h->sg_on_dev != on_device || h->sg_maps != h->d_maps || h->sg_traj != h->d_traj ||
                       h->sg_noise != (const void*)h->noise_all || h->sg_frames != frames_key;
  std::vector<LaunchRec> recs;
  int rc;
  if (rebuild) {
    if (h->sgx) cudaGraphExecDestroy(h->sgx);
    if (h->sg) cudaGraphDestroy(h->sg);
    h->sgx = nullptr;
    h->sg = nullptr;
    if (h->philox && (rc = h->phx.reserve(2 * h->K, h->err))) return rc;  // no allocation while capturing
    h->rec = &recs;
    h->rec_only = false;
    PF_CUDA(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal), h->err);
    auto fail = [&](int code) {
      h->rec = nullptr;
      cudaGraph_t g = nullptr;
      cudaStreamEndCapture(h->stream, &g);
      if (g) cudaGraphDestroy(g);
      return code;
    };
    if (!on_device && cudaMemcpyAsync(h->d_frames, h->h_stage, (size_t)h->n_videos * h->H * h->W,
                                      cudaMemcpyHostToDevice, h->stream) != cudaSuccess)
      return fail(PF_ECUDA);
    if ((rc = launch_maps(h, dframes, 1))) return fail(rc);
    if (h->philox && (rc = h->phx.draw(h->stream, 2 * h->K, h->noise_all, h->u_all, h->err))) return fail(rc);
    if ((rc = launch_frame(h, h->d_maps, (long long)map_elems, 0, 1))) return fail(rc);
    h->rec = nullptr;
    PF_CUDA(cudaStreamEndCapture(h->stream, &h->sg), h->err);
    PF_CUDA(cudaGraphInstantiate(&h->sgx, h->sg, 0), h->err);
    if (recs.size() != 3) {
      h->err = "step graph: unexpected launch sequence";
      return PF_ECUDA;
    }
    size_t n = 0;
    PF_CUDA(cudaGraphGetNodes(h->sg, nullptr, &n), h->err);
    std::vector<cudaGraphNode_t> nodes(n);
    PF_CUDA(cudaGraphGetNodes(h->sg, nodes.data(), &n), h->err);
    for (auto& nd : h->sg_node) nd = nullptr;
    for (cudaGraphNode_t nd : nodes) {
      cudaGraphNodeType ty;
      PF_CUDA(cudaGraphNodeGetType(nd, &ty), h->err);
      if (ty != cudaGraphNodeTypeKernel) continue;
      cudaKernelNodeParams kp{};
      PF_CUDA(cudaGraphKernelNodeGetParams(nd, &kp), h->err);
      for (int i = 0; i < 3; ++i)
        if (kp.func == recs[i].fn) h->sg_node[i] = nd;
    }
    if (!h->sg_node[0] || !h->sg_node[1] || !h->sg_node[2]) {
      h->err = "step graph: kernel nodes not found";
      return PF_ECUDA;
    }
    h->sg_on_dev = on_device;
    h->sg_maps = h->d_maps;
    h->sg_traj = h->d_traj;
    h->sg_noise = h->noise_all;
    h->sg_frames = frames_key;
  } else {
    h->rec = &recs;
    h->rec_only = true;  // arguments only (the Philox draws' arguments never change)
    rc = launch_maps(h, dframes, 1);
    if (!rc) rc = launch_frame(h, h->d_maps, (long long)map_elems, 0, 1);
    h->rec = nullptr;
    h->rec_only = false;
    if (rc) return rc;
    for (int i = 0; i < 3; ++i) {
      cudaKernelNodeParams kp{};
      kp.func = const_cast<void*>(recs[i].fn);
      kp.gridDim = recs[i].grid;
      kp.blockDim = recs[i].block;
      kp.sharedMemBytes = (unsigned)recs[i].smem;
      void* args[1] = {recs[i].args.data()};
      kp.kernelParams = args;
      PF_CUDA(cudaGraphExecKernelNodeSetParams(h->sgx, h->sg_node[i], &kp), h->err);
    }
  }
  PF_CUDA(cudaGraphLaunch(h->sgx, h->stream), h->err);
  if (h->philox) h->launches += 4;
  return PF_OK;
}

static int run_complete(pf_handle* h);
static int run_enqueue(pf_handle* h, const uint8_t* frames, int32_t F, int32_t on_device, double* traj_out,
                       cudaStream_t ext, bool sync_call = false) {
  if (!h || !frames || F < 1 || !traj_out) return PF_EINVAL;
  if (h->n_shards > 1) {
    h->err = "sharded handle: drive frames with pf_shard_*";
    return PF_EINVAL;
  }
  PF_CUDA(cudaSetDevice(h->device), h->err);
  if (ext) {
    if (!h->xin) {
      PF_CUDA(cudaEventCreateWithFlags(&h->xin, cudaEventDisableTiming), h->err);
      PF_CUDA(cudaEventCreateWithFlags(&h->xout, cudaEventDisableTiming), h->err);
    }
    PF_CUDA(cudaEventRecord(h->xin, ext), h->err);  // the caller's producers of `frames`
    PF_CUDA(cudaStreamWaitEvent(h->stream, h->xin, 0), h->err);
  }
  h->launches = 0;
  const size_t fbytes = (size_t)h->n_videos * F * h->H * h->W;
  const size_t map_elems = (size_t)h->Hm * h->Wm;
  int rc;
  if ((rc = grow((void**)&h->d_maps, &h->maps_cap, (size_t)h->n_videos * F * map_elems * h->rs, h->err))) return rc;
  if ((rc = grow((void**)&h->d_traj, &h->traj_cap, (size_t)h->n_tracks * F * 2 * 8, h->err))) return rc;
  if (h->tracing) {
    const size_t need = (size_t)F * (h->n_tiles + h->n_chunks) * 8 * 8;
    if (h->trace_cap < need) h->g_F = -1;  // re-capture with the new buffer
    if ((rc = grow((void**)&h->d_trace, &h->trace_cap, need, h->err))) return rc;
    PF_CUDA(cudaMemsetAsync(h->d_trace, 0, need, h->stream), h->err);
  }
  if (h->profiling) {
    while ((int)h->pev.size() < 3 * F) {
      cudaEvent_t e;
      PF_CUDA(cudaEventCreate(&e), h->err);
      h->pev.push_back(e);
    }
  }
  const uint8_t* dframes = frames;
  if (!on_device) {
    if ((rc = grow((void**)&h->d_frames, &h->frames_cap, fbytes, h->err))) return rc;
    dframes = h->d_frames;
  }
  // a synchronous one-frame step into host memory: zero-copy result
  // (any synchronous run into host memory: the tile tables write the
  // trajectory and the degeneracy flags into host-mapped memory)
  h->zc_step = sync_call && !h->split_table && h->n_shards == 1 && !h->profiling &&
               std::getenv("PF_NO_ZC_STEP") == nullptr;
  if (h->zc_step) {
    cudaPointerAttributes at{};
    const bool host_dst = cudaPointerGetAttributes(&at, traj_out) != cudaSuccess || at.type != cudaMemoryTypeDevice;
    cudaGetLastError();
    h->zc_step = host_dst;
  }
  if (h->zc_step) {
    const size_t need = (size_t)h->n_tracks * F * 2 * 8;
    if (h->est_map_cap < need) {
      if (h->pending) {
        const int prc = run_complete(h);
        if (prc) return prc;
      }
      PF_CUDA(cudaStreamSynchronize(h->stream), h->err);
      if (h->h_est_map) cudaFreeHost(h->h_est_map);
      h->h_est_map = nullptr;
      h->est_map_cap = 0;
      PF_CUDA(cudaHostAlloc(&h->h_est_map, need, cudaHostAllocMapped), h->err);
      h->est_map_cap = need;
      PF_CUDA(cudaHostGetDevicePointer(&h->d_est_map, h->h_est_map, 0), h->err);
    }
    if (!h->h_deg_map) {
      PF_CUDA(cudaHostAlloc(&h->h_deg_map, (size_t)h->n_tracks * sizeof(int), cudaHostAllocMapped), h->err);
      PF_CUDA(cudaHostGetDevicePointer(&h->d_deg_map, h->h_deg_map, 0), h->err);
    }
    if (h->pending) {  // the flags below are the previous run's until it completes (its error is reported here)
      const int prc = run_complete(h);
      if (prc) return prc;
    }
    for (int i = 0; i < h->n_tracks; ++i) h->h_deg_map[i] = INT_MAX;
  }
  PF_CUDA(cudaEventRecord(h->ev[0], h->stream), h->err);
  // per-frame steps: one graph launch (stage timings collapse to "frames")
  const bool step_graph = F == 1 && h->use_graphs && !h->profiling && !h->tracing && !h->dbg_anc &&
                          !h->split_table && (on_device || (sync_call && fbytes <= kStageBytes));
  if (step_graph) {
    if (!on_device) {
      if (!h->h_stage) PF_CUDA(cudaMallocHost(&h->h_stage, kStageBytes), h->err);
      PF_CUDA(cudaStreamSynchronize(h->stream), h->err);  // the staging buffer's previous copy is done
      std::memcpy(h->h_stage, frames, fbytes);
    }
    if (h->philox) {
      if ((rc = grow((void**)&h->noise_all, &h->noise_cap, (size_t)2 * h->K * 8, h->err))) return rc;
      if ((rc = grow((void**)&h->u_all, &h->u_cap, 8, h->err))) return rc;
    }
    PF_CUDA(cudaEventRecord(h->ev[1], h->stream), h->err);
    PF_CUDA(cudaEventRecord(h->ev[2], h->stream), h->err);
    if ((rc = step_graph_launch(h, dframes, on_device))) return rc;
  } else {
  // (C3's 100 MB: 31.4 -> 30.0 ms per step; below ~8 MB the extra map launches
  // cost more than the upload they hide -- C2's 1.6 MB: +0.1 ms)
  if (!on_device && h->n_videos == 1 && F >= kUploadChunks && fbytes >= (8u << 20)) {
    // chunked upload on the copy stream; each chunk's maps start when it lands
    // ("upload" then times only the exposed first chunk)
    if (!h->cstream) {
      PF_CUDA(cudaStreamCreateWithFlags(&h->cstream, cudaStreamNonBlocking), h->err);
      for (auto& e : h->cev) PF_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), h->err);
    }
    PF_CUDA(cudaStreamWaitEvent(h->cstream, h->ev[0], 0), h->err);  // earlier readers of d_frames
    const size_t fb = (size_t)h->H * h->W;
    const int per = (F + kUploadChunks - 1) / kUploadChunks;
    for (int c = 0; c * per < F; ++c) {
      const int f0 = c * per, nf = std::min(per, F - f0);
      PF_CUDA(cudaMemcpyAsync(h->d_frames + f0 * fb, frames + f0 * fb, nf * fb, cudaMemcpyHostToDevice, h->cstream),
              h->err);
      PF_CUDA(cudaEventRecord(h->cev[c], h->cstream), h->err);
    }
    for (int c = 0; c * per < F; ++c) {
      const int f0 = c * per, nf = std::min(per, F - f0);
      PF_CUDA(cudaStreamWaitEvent(h->stream, h->cev[c], 0), h->err);
      if (c == 0) PF_CUDA(cudaEventRecord(h->ev[1], h->stream), h->err);
      if ((rc = launch_maps(h, dframes, F, f0, nf))) return rc;
    }
  } else {
    if (!on_device) {
      const uint8_t* src = frames;
      if (sync_call && fbytes <= kStageBytes && is_pageable(frames)) {  // small host frames: pinned staging
        if (!h->h_stage) PF_CUDA(cudaMallocHost(&h->h_stage, kStageBytes), h->err);
        PF_CUDA(cudaStreamSynchronize(h->stream), h->err);  // the staging buffer's previous copy is done
        std::memcpy(h->h_stage, frames, fbytes);
        src = h->h_stage;
      }
      PF_CUDA(cudaMemcpyAsync(h->d_frames, src, fbytes, cudaMemcpyHostToDevice, h->stream), h->err);
    }
    PF_CUDA(cudaEventRecord(h->ev[1], h->stream), h->err);
    if ((rc = launch_maps(h, dframes, F))) return rc;
  }
  if (h->philox) {  // the reference stream's draws of every frame: 2K normals, then random()
    if ((rc = grow((void**)&h->noise_all, &h->noise_cap, (size_t)F * 2 * h->K * 8, h->err))) return rc;
    if ((rc = grow((void**)&h->u_all, &h->u_cap, (size_t)F * 8, h->err))) return rc;
    for (int f = 0; f < F; ++f)
      if ((rc = h->phx.draw(h->stream, 2 * h->K, h->noise_all + (size_t)f * 2 * h->K, h->u_all + f, h->err)))
        return rc;
    h->launches += 4LL * F;
  }
  PF_CUDA(cudaEventRecord(h->ev[2], h->stream), h->err);
  const long long vstride = (long long)F * map_elems;  // elements between videos
  const bool graph_ok = h->use_graphs && !h->profiling && F >= 4;
  if (graph_ok && h->gexec && h->g_start == h->frame_counter && h->g_cur == h->cur && h->g_F == F &&
      h->g_maps == h->d_maps && h->g_traj == h->d_traj && h->g_ident == h->ident_next &&
      h->g_noise == (const void*)h->noise_all && h->g_est == (h->zc_step ? (const void*)h->d_est_map : nullptr)) {
    PF_CUDA(cudaGraphLaunch(h->gexec, h->stream), h->err);
    h->ident_next = false;
    h->frame_counter += F;
    if (F % 2) h->cur = 1 - h->cur;
    h->launches += 2LL * F;
  } else if (graph_ok) {
    const long long start = h->frame_counter;
    const int cur0 = h->cur;
    const bool ident0 = h->ident_next;
    cudaGraph_t g = nullptr;
    PF_CUDA(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal), h->err);
    for (int f = 0; f < F; ++f) {
      const char* slot = (const char*)h->d_maps + (size_t)f * map_elems * h->rs;
      if ((rc = launch_frame(h, slot, vstride, f, F))) {
        cudaStreamEndCapture(h->stream, &g);
        if (g) cudaGraphDestroy(g);
        return rc;
      }
    }
    PF_CUDA(cudaStreamEndCapture(h->stream, &g), h->err);
    if (h->gexec) cudaGraphExecDestroy(h->gexec);
    h->gexec = nullptr;
    PF_CUDA(cudaGraphInstantiate(&h->gexec, g, 0), h->err);
    cudaGraphDestroy(g);
    h->g_start = start;
    h->g_cur = cur0;
    h->g_ident = ident0;
    h->g_noise = h->noise_all;
    h->g_F = F;
    h->g_maps = h->d_maps;
    h->g_traj = h->d_traj;
    h->g_est = h->zc_step ? (const void*)h->d_est_map : nullptr;
    PF_CUDA(cudaGraphLaunch(h->gexec, h->stream), h->err);
  } else {
    for (int f = 0; f < F; ++f) {
      const char* slot = (const char*)h->d_maps + (size_t)f * map_elems * h->rs;
      if ((rc = launch_frame(h, slot, vstride, f, F))) return rc;
    }
  }
  }  // not a step graph
  PF_CUDA(cudaEventRecord(h->ev[3], h->stream), h->err);
  // device or (pinned / pageable) host destination; a synchronous call with a
  // pageable destination lands in pinned memory and is copied out after the sync
  const size_t tbytes = (size_t)h->n_tracks * F * 2 * 8;
  h->traj_user = nullptr;
  h->zc_pending = false;
  if (h->zc_step) {  // the estimate is already on its way into host-mapped memory
    h->zc_step = false;
    h->zc_pending = true;
    h->traj_user = traj_out;
    h->traj_bytes = tbytes;
    PF_CUDA(cudaEventRecord(h->ev[4], h->stream), h->err);
    h->pending = true;
    h->pending_F = F;
    return PF_OK;
  }
  if (sync_call && is_pageable(traj_out)) {
    if (h->h_traj_cap < tbytes) {
      if (h->h_traj) cudaFreeHost(h->h_traj);
      h->h_traj = nullptr;
      h->h_traj_cap = 0;
      PF_CUDA(cudaMallocHost(&h->h_traj, tbytes), h->err);
      h->h_traj_cap = tbytes;
    }
    PF_CUDA(cudaMemcpyAsync(h->h_traj, h->d_traj, tbytes, cudaMemcpyDeviceToHost, h->stream), h->err);
    h->traj_user = traj_out;
    h->traj_bytes = tbytes;
  } else {
    PF_CUDA(cudaMemcpyAsync(traj_out, h->d_traj, tbytes, cudaMemcpyDefault, h->stream), h->err);
  }
  if ((rc = queue_degenerate(h))) return rc;
  PF_CUDA(cudaEventRecord(h->ev[4], h->stream), h->err);
  if (ext) {  // the caller's later work sees the trajectory
    PF_CUDA(cudaEventRecord(h->xout, h->stream), h->err);
    PF_CUDA(cudaStreamWaitEvent(ext, h->xout, 0), h->err);
  }
  h->pending = true;
  h->pending_F = F;
  return PF_OK;
}

// stage timings of the last completed run from its events (on demand: the
// elapsed-time queries cost the per-frame step a few microseconds)
static void compute_timings(pf_handle* h) {
  if (!h->timings_stale || h->pending) return;
  h->timings_stale = false;
  const int F = h->timings_F;
  float ms;
  cudaEventElapsedTime(&ms, h->ev[0], h->ev[4]);
  h->timings[0] = ms;
  cudaEventElapsedTime(&ms, h->ev[0], h->ev[1]);
  h->timings[1] = ms;
  cudaEventElapsedTime(&ms, h->ev[1], h->ev[2]);
  h->timings[2] = ms;
  cudaEventElapsedTime(&ms, h->ev[2], h->ev[3]);
  h->timings[3] = ms;
  h->timings[4] = 0.f;
  if (h->profiling) {
    float fsum = 0.f, tsum = 0.f;
    for (int f = 0; f < F; ++f) {
      cudaEventElapsedTime(&ms, h->pev[3 * f], h->pev[3 * f + 1]);
      fsum += ms;
      cudaEventElapsedTime(&ms, h->pev[3 * f + 1], h->pev[3 * f + 2]);
      tsum += ms;
    }
    h->timings[3] = fsum;
    h->timings[4] = tsum;
  }
  cudaEventElapsedTime(&ms, h->ev[3], h->ev[4]);
  h->timings[5] = ms;
}

// wait for the enqueued run; timings and the degeneracy check
static int run_complete(pf_handle* h) {
  if (!h->pending) return PF_OK;
  PF_CUDA(cudaSetDevice(h->device), h->err);
  PF_CUDA(cudaStreamSynchronize(h->stream), h->err);
  h->pending = false;
  const int F = h->pending_F;
  if (h->zc_pending) {
    std::memcpy(h->traj_user, h->h_est_map, h->traj_bytes);
    h->traj_user = nullptr;
  } else if (h->traj_user) {
    std::memcpy(h->traj_user, h->h_traj, h->traj_bytes);
    h->traj_user = nullptr;
  }
  if (h->philox) {
    const int rc = h->phx.check(h->err);
    if (rc) return rc;
  }
  h->timings_stale = true;  // event times read on demand (pf_last_timings)
  h->timings_F = F;
  if (h->zc_pending) {
    h->zc_pending = false;
    int m = INT_MAX;
    for (int i = 0; i < h->n_tracks; ++i) m = std::min(m, h->h_deg_map[i]);
    if (m != INT_MAX) {
      h->degenerate_frame = m;
      h->err = "weight sum degenerated (frame " + std::to_string(m) + ")";
      return PF_EDEGENERATE;
    }
    return PF_OK;
  }
  return finish_degenerate(h);
}

int pf_run(pf_handle* h, const uint8_t* frames, int32_t F, int32_t on_device, double* traj_out) {
  int rc = run_enqueue(h, frames, F, on_device, traj_out, nullptr, true);
  if (rc) return rc;
  return run_complete(h);
}

int pf_run_async(pf_handle* h, const uint8_t* frames, int32_t F, int32_t on_device, double* traj_out,
                 void* stream) {
  return run_enqueue(h, frames, F, on_device, traj_out, (cudaStream_t)stream);
}

int pf_step_async(pf_handle* h, const uint8_t* frame, int32_t on_device, double* est_out, void* stream) {
  return run_enqueue(h, frame, 1, on_device, est_out, (cudaStream_t)stream);
}

int pf_stream_wait(pf_handle* h, void* stream) {
  if (!h) return PF_EINVAL;
  if (!stream) return PF_OK;
  PF_CUDA(cudaSetDevice(h->device), h->err);
  if (!h->xin) {
    PF_CUDA(cudaEventCreateWithFlags(&h->xin, cudaEventDisableTiming), h->err);
    PF_CUDA(cudaEventCreateWithFlags(&h->xout, cudaEventDisableTiming), h->err);
  }
  PF_CUDA(cudaEventRecord(h->xin, (cudaStream_t)stream), h->err);
  PF_CUDA(cudaStreamWaitEvent(h->stream, h->xin, 0), h->err);
  return PF_OK;
}

int pf_sync(pf_handle* h) {
  if (!h) return PF_EINVAL;
  return run_complete(h);
}

int pf_likelihood_maps(pf_handle* h, const uint8_t* frames, int32_t F, void* maps_out) {
  if (!h || !frames || F < 1 || !maps_out || h->n_videos != 1) return PF_EINVAL;
  PF_CUDA(cudaSetDevice(h->device), h->err);
  const size_t fbytes = (size_t)F * h->H * h->W;
  const size_t mbytes = (size_t)F * h->Hm * h->Wm * h->rs;
  int rc;
  if ((rc = grow((void**)&h->d_frames, &h->frames_cap, fbytes, h->err))) return rc;
  if ((rc = grow((void**)&h->d_maps, &h->maps_cap, mbytes, h->err))) return rc;
  h->g_F = -1;  // the map buffer may have moved: re-capture the frame graph
  PF_CUDA(cudaMemcpyAsync(h->d_frames, frames, fbytes, cudaMemcpyHostToDevice, h->stream), h->err);
  if ((rc = launch_maps(h, h->d_frames, F))) return rc;
  PF_CUDA(cudaMemcpyAsync(maps_out, h->d_maps, mbytes, cudaMemcpyDeviceToHost, h->stream), h->err);
  PF_CUDA(cudaStreamSynchronize(h->stream), h->err);
  return PF_OK;
}

int pf_step(pf_handle* h, const uint8_t* frame, int32_t on_device, double* est_out) {
  return pf_run(h, frame, 1, on_device, est_out);
}

int pf_degenerate_frame(const pf_handle* h) { return h ? h->degenerate_frame : -1; }

int pf_set_profiling(pf_handle* h, int32_t on) {
  if (!h) return PF_EINVAL;
  h->profiling = on != 0;
  return PF_OK;
}

int pf_set_trace(pf_handle* h, int32_t on) {
  if (!h) return PF_EINVAL;
  if ((on != 0) != h->tracing) h->g_F = -1;  // kernel arguments change: re-capture
  h->tracing = on != 0;
  return PF_OK;
}

int pf_get_trace(pf_handle* h, uint64_t* out, int64_t n) {
  if (!h || !out || n < 0) return PF_EINVAL;
  PF_CUDA(cudaSetDevice(h->device), h->err);
  PF_CUDA(cudaStreamSynchronize(h->stream), h->err);
  if ((size_t)n * 8 > h->trace_cap) return PF_EINVAL;
  PF_CUDA(cudaMemcpy(out, h->d_trace, (size_t)n * 8, cudaMemcpyDeviceToHost), h->err);
  return PF_OK;
}

int pf_last_timings(const pf_handle* h, float* ms6) {
  if (!h || !ms6) return PF_EINVAL;
  compute_timings(const_cast<pf_handle*>(h));
  for (int i = 0; i < 6; ++i) ms6[i] = h->timings[i];
  return PF_OK;
}
int64_t pf_last_launches(const pf_handle* h) { return h ? h->launches : -1; }

int pf_get_state(pf_handle* h, int32_t track, void* xs, void* ys, void* cdf) {
  if (!h || track < 0 || track >= h->n_tracks) return PF_EINVAL;
  PF_CUDA(cudaSetDevice(h->device), h->err);
  PF_CUDA(cudaStreamSynchronize(h->stream), h->err);
  const size_t K = (size_t)h->Kl;
  std::vector<unsigned char> buf(K * h->vs);
  PF_CUDA(cudaMemcpy(buf.data(), (char*)h->X[h->cur] + track * K * h->vs, K * h->vs, cudaMemcpyDeviceToHost), h->err);
  for (size_t k = 0; k < K; ++k) {
    if (xs) std::memcpy((char*)xs + k * h->rs, buf.data() + k * h->vs, h->rs);
    if (ys) std::memcpy((char*)ys + k * h->rs, buf.data() + k * h->vs + h->rs, h->rs);
  }
  if (cdf)
    PF_CUDA(cudaMemcpy(cdf, (char*)h->C[h->cur] + track * K * h->rs, K * h->rs, cudaMemcpyDeviceToHost), h->err);
  return PF_OK;
}

int pf_set_rng_philox(pf_handle* h, const uint64_t* state11) {
  if (!h || !state11) return PF_EINVAL;
  if (h->n_tracks != 1 || h->n_shards != 1 || h->split_table) {
    h->err = "rng='numpy-philox' needs a single unsharded track";
    return PF_EINVAL;
  }
  if (h->tpb != 128 && h->tpb != 256) {
    h->err = "rng='numpy-philox' runs at 128 or 256 threads per block";
    return PF_EINVAL;
  }
  PF_CUDA(cudaSetDevice(h->device), h->err);
  if (h->pending) run_complete(h);
  PF_CUDA(cudaStreamSynchronize(h->stream), h->err);
  int rc = h->phx.init(state11, h->err);
  if (rc) return rc;
  h->philox = true;
  h->g_F = -1;
  PF_CUDA(set_fused_smem(h), h->err);
  PF_CUDA(cudaDeviceSynchronize(), h->err);
  return PF_OK;
}

int pf_set_state(pf_handle* h, int32_t track, const void* xs, const void* ys, int64_t frame) {
  if (!h || track < 0 || track >= h->n_tracks || !xs || !ys || frame < 0 || frame > INT_MAX) return PF_EINVAL;
  if (h->n_shards > 1) {
    h->err = "pf_set_state: sharded handles are not supported";
    return PF_EINVAL;
  }
  PF_CUDA(cudaSetDevice(h->device), h->err);
  if (h->pending) {
    const int rc = run_complete(h);
    if (rc && rc != PF_EDEGENERATE) return rc;
  }
  PF_CUDA(cudaStreamSynchronize(h->stream), h->err);
  const size_t K = (size_t)h->Kl;
  std::vector<unsigned char> buf(K * h->vs);
  for (size_t k = 0; k < K; ++k) {
    std::memcpy(buf.data() + k * h->vs, (const char*)xs + k * h->rs, h->rs);
    std::memcpy(buf.data() + k * h->vs + h->rs, (const char*)ys + k * h->rs, h->rs);
  }
  PF_CUDA(cudaMemcpy((char*)h->X[h->cur] + track * K * h->vs, buf.data(), K * h->vs, cudaMemcpyHostToDevice), h->err);
  // every track enters frame `frame` with identity ancestors; the table-ready
  // counters restart at the value frame `frame`'s successor expects
  h->frame_counter = frame;
  h->ident_next = true;
  std::vector<unsigned long long> sync((size_t)h->n_tracks * 4, 0ULL);
  for (int i = 0; i < h->n_tracks; ++i) sync[(size_t)i * 4 + 1] = (unsigned long long)h->n_chunks * (unsigned long long)frame;
  PF_CUDA(cudaMemcpy(h->tsync, sync.data(), sync.size() * 8, cudaMemcpyHostToDevice), h->err);
  return PF_OK;
}

int pf_get_debug(pf_handle* h, int32_t track, int64_t* anc, void* loglik) {
  if (!h || track < 0 || track >= h->n_tracks) return PF_EINVAL;
  PF_CUDA(cudaSetDevice(h->device), h->err);
  const size_t K = (size_t)h->Kl, KT = K * h->n_tracks;
  if (!h->dbg_anc) {
    // enable debug capture for subsequent frames
    PF_CUDA(cudaMalloc(&h->dbg_anc, KT * 8), h->err);
    PF_CUDA(cudaMalloc(&h->dbg_L, KT * h->rs), h->err);
    h->g_F = -1;  // captured graphs do not write the debug buffers
    return PF_OK;
  }
  PF_CUDA(cudaStreamSynchronize(h->stream), h->err);
  if (anc) PF_CUDA(cudaMemcpy(anc, h->dbg_anc + track * K, K * 8, cudaMemcpyDeviceToHost), h->err);
  if (loglik)
    PF_CUDA(cudaMemcpy(loglik, (char*)h->dbg_L + track * K * h->rs, K * h->rs, cudaMemcpyDeviceToHost), h->err);
  return PF_OK;
}

// ---------------------------------------------------------------------------
// input side: device video rendering, PFVD ingest
// ---------------------------------------------------------------------------
// model._reflect (model.py:105-121): one step with specular bounces
static void reflect_step(double& v, double& d, double hi) {
  v += d;
  while (v < 0.0 || v > hi) {
    if (v < 0.0) {
      v = -v;
      d = -d;
    }
    if (v > hi) {
      v = 2.0 * hi - v;
      d = -d;
    }
  }
}

int pf_generate_video(const pf_params* params, int32_t F, int32_t W, int32_t H, double x0, double y0,
                      uint64_t seed, const int32_t* offsets_xy, int32_t n_off, uint8_t* frames_dev,
                      double* truth_host, int32_t device) {
  if (!params || F < 1 || W < 1 || H < 1 || n_off < 1 || !offsets_xy || !frames_dev || !truth_host) {
    g_err = "bad video arguments";
    return PF_EINVAL;
  }
  if (F < 1) {
    g_err = "frames must be at least 1";
    return PF_EINVAL;
  }
  if (!(x0 >= 0.0 && x0 <= W - 1 && y0 >= 0.0 && y0 <= H - 1)) {
    g_err = "start outside frame bounds";
    return PF_EINVAL;
  }
  if ((W == 1 && params->drift_x != 0.0) || (H == 1 && params->drift_y != 0.0)) {
    g_err = "a 1-pixel frame axis with non-zero drift has no bounded trajectory";
    return PF_EINVAL;  // (the reference's bounce loop would never end)
  }
  PF_CUDA(cudaSetDevice(device), g_err);
  int rc = init_device_tables(device, g_err);
  if (rc) return rc;
  // truth trajectory and the clipped disk pixels per frame (model.py:136-155)
  std::vector<int> fg((size_t)F * n_off);
  double x = x0, y = y0, dx = params->drift_x, dy = params->drift_y;
  for (int t = 0; t < F; ++t) {
    truth_host[2 * t] = x;
    truth_host[2 * t + 1] = y;
    const long cx = (long)std::nearbyint(x), cy = (long)std::nearbyint(y);  // round half to even
    for (int j = 0; j < n_off; ++j) {
      const long col = std::min(std::max(offsets_xy[2 * j] + cx, 0L), (long)W - 1);
      const long row = std::min(std::max(offsets_xy[2 * j + 1] + cy, 0L), (long)H - 1);
      fg[(size_t)t * n_off + j] = (int)(row * W + col);
    }
    reflect_step(x, dx, W - 1.0);
    reflect_step(y, dy, H - 1.0);
  }
  int* d_fg = nullptr;
  PF_CUDA(cudaMalloc(&d_fg, fg.size() * sizeof(int)), g_err);
  cudaError_t ce = cudaMemcpy(d_fg, fg.data(), fg.size() * sizeof(int), cudaMemcpyHostToDevice);
  const long long frame_px = (long long)W * H, n = frame_px * F;
  const unsigned long long xs = pfv::video_stream_state(seed);
  if (ce == cudaSuccess) {
    const long long threads = (n + 7) / 8;
    pfv::render_background<<<(unsigned)((threads + 255) / 256), 256>>>(frames_dev, n, xs, params->bg_mean,
                                                                         params->noise_std);
    pfv::render_object<<<F, 128>>>(frames_dev, d_fg, n_off, frame_px, xs, params->fg_mean, params->noise_std);
    ce = cudaDeviceSynchronize();
  }
  cudaFree(d_fg);
  PF_CUDA(ce, g_err);
  return PF_OK;
}

// PFVD container: "PFVD", u32 frames, width, height, pixels (model.py:274-297)
int pf_pfvd_info(const char* path, int32_t* fwh) {
  if (!path || !fwh) return PF_EINVAL;
  FILE* fh = std::fopen(path, "rb");
  if (!fh) {
    g_err = std::string(path) + ": cannot open";
    return PF_EIO;
  }
  char magic[4];
  uint32_t hdr[3];
  const size_t m = std::fread(magic, 1, 4, fh);
  if (m != 4 || std::memcmp(magic, "PFVD", 4) != 0) {
    std::fclose(fh);
    g_err = std::string(path) + ": bad container magic at offset 0";
    return PF_EIO;
  }
  if (std::fread(hdr, 4, 3, fh) != 3) {
    std::fclose(fh);
    g_err = std::string(path) + ": truncated header at offset 4";
    return PF_EIO;
  }
  std::fseek(fh, 0, SEEK_END);
  const long long payload = (long long)std::ftell(fh) - 16;
  std::fclose(fh);
  const long long expected = (long long)hdr[0] * hdr[1] * hdr[2];
  if (payload != expected) {
    g_err = std::string(path) + ": expected " + std::to_string(expected) + " pixel bytes at offset 16, got " +
            std::to_string(payload);
    return PF_EIO;
  }
  fwh[0] = (int32_t)hdr[0];
  fwh[1] = (int32_t)hdr[1];
  fwh[2] = (int32_t)hdr[2];
  return PF_OK;
}

// streams the payload through two pinned staging buffers into device memory
// (the read of chunk i+1 overlaps the copy of chunk i)
int pf_read_pfvd(const char* path, uint8_t* frames_dev, int64_t capacity, int32_t* fwh, int32_t device) {
  if (!frames_dev || !fwh) return PF_EINVAL;
  int rc = pf_pfvd_info(path, fwh);
  if (rc) return rc;
  const long long total = (long long)fwh[0] * fwh[1] * fwh[2];
  if (total > capacity) {
    g_err = "device buffer too small for the video";
    return PF_EINVAL;
  }
  PF_CUDA(cudaSetDevice(device), g_err);
  FILE* fh = std::fopen(path, "rb");
  if (!fh) {
    g_err = std::string(path) + ": cannot open";
    return PF_EIO;
  }
  std::fseek(fh, 16, SEEK_SET);
  const size_t chunk = 8u << 20;
  uint8_t* pin[2] = {nullptr, nullptr};
  cudaEvent_t done[2] = {nullptr, nullptr};
  cudaStream_t st = nullptr;
  cudaError_t ce = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  for (int i = 0; i < 2 && ce == cudaSuccess; ++i) {
    ce = cudaMallocHost(&pin[i], chunk);
    if (ce == cudaSuccess) ce = cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming);
  }
  long long off = 0;
  int k = 0;
  while (ce == cudaSuccess && off < total) {
    const size_t n = (size_t)std::min<long long>(chunk, total - off);
    ce = cudaEventSynchronize(done[k]);  // the previous copy out of this staging buffer is done
    if (ce != cudaSuccess) break;
    if (std::fread(pin[k], 1, n, fh) != n) {
      g_err = std::string(path) + ": short read";
      ce = cudaErrorUnknown;
      break;
    }
    ce = cudaMemcpyAsync(frames_dev + off, pin[k], n, cudaMemcpyHostToDevice, st);
    if (ce == cudaSuccess) ce = cudaEventRecord(done[k], st);
    off += (long long)n;
    k ^= 1;
  }
  if (ce == cudaSuccess) ce = cudaStreamSynchronize(st);
  std::fclose(fh);
  for (int i = 0; i < 2; ++i) {
    if (pin[i]) cudaFreeHost(pin[i]);
    if (done[i]) cudaEventDestroy(done[i]);
  }
  if (st) cudaStreamDestroy(st);
  if (ce != cudaSuccess) {
    if (g_err.empty() || g_err.find("short read") == std::string::npos)
      g_err = std::string("CUDA error ") + cudaGetErrorString(ce) + " reading PFVD";
    return g_err.find("short read") != std::string::npos ? PF_EIO : PF_ECUDA;
  }
  return PF_OK;
}

// ---------------------------------------------------------------------------
// sharded filter: one track split by particle range over
// n_shards handles; the host runs the three per-frame exchanges (NCCL
// all-gathers on the handle's stream, or pf_shard_local_allgather for shards
// that share a process)
// ---------------------------------------------------------------------------
int pf_shard_create(pf_handle** out, const pf_config* cfg, int32_t n_shards, int32_t shard) {
  return create_impl(out, cfg, n_shards, shard);
}

int pf_shard_info(const pf_handle* h, int64_t* out4) {
  if (!h || !out4) return PF_EINVAL;
  out4[0] = h->shard_tiles;
  out4[1] = h->tile0;
  out4[2] = h->nl;
  out4[3] = h->Kl;
  return PF_OK;
}

int pf_shard_buffers(pf_handle* h, void** out8) {
  if (!h || !out8) return PF_EINVAL;
  for (int i = 0; i < 8; ++i) out8[i] = h->peer[h->shard][i];
  return PF_OK;
}

int pf_shard_ipc_export(pf_handle* h, void* out) {
  if (!h || !out) return PF_EINVAL;
  PF_CUDA(cudaSetDevice(h->device), h->err);
  cudaIpcMemHandle_t* o = reinterpret_cast<cudaIpcMemHandle_t*>(out);
  for (int i = 0; i < 8; ++i) PF_CUDA(cudaIpcGetMemHandle(&o[i], h->peer[h->shard][i]), h->err);
  return PF_OK;
}

// direct peer access from h's device to `peer_dev` (the fused kernel reads
// remote source tiles, the finish kernel stores remote window records)
static int enable_peer(pf_handle* h, int peer_dev) {
  if (peer_dev == h->device) return PF_OK;
  int can = 0;
  PF_CUDA(cudaDeviceCanAccessPeer(&can, h->device, peer_dev), h->err);
  if (!can) {
    h->err = "device " + std::to_string(h->device) + " cannot access device " + std::to_string(peer_dev) +
             " peer-to-peer (NVLink / PCIe P2P required for a shard on another GPU)";
    return PF_EINVAL;
  }
  PF_CUDA(cudaSetDevice(h->device), h->err);
  const cudaError_t e = cudaDeviceEnablePeerAccess(peer_dev, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();  // not an error: clear it
  } else if (e != cudaSuccess) {
    h->err = std::string("cudaDeviceEnablePeerAccess: ") + cudaGetErrorString(e);
    return PF_ECUDA;
  }
  return PF_OK;
}

int pf_shard_set_peer(pf_handle* h, int32_t peer, void* const* ptrs8) {
  if (!h || !ptrs8 || peer < 0 || peer >= h->n_shards || peer == h->shard) return PF_EINVAL;
  for (int i = 0; i < 8; ++i) {
    cudaPointerAttributes at{};
    if (!ptrs8[i] || cudaPointerGetAttributes(&at, ptrs8[i]) != cudaSuccess || at.type != cudaMemoryTypeDevice) {
      cudaGetLastError();
      h->err = "pf_shard_set_peer: peer buffer " + std::to_string(i) + " is not device memory";
      return PF_EINVAL;
    }
    const int rc = enable_peer(h, at.device);
    if (rc) return rc;
  }
  for (int i = 0; i < 8; ++i) h->peer[peer][i] = ptrs8[i];
  return PF_OK;
}

int pf_shard_open_peer(pf_handle* h, int32_t peer, const void* handles) {
  if (!h || !handles || peer < 0 || peer >= h->n_shards || peer == h->shard) return PF_EINVAL;
  PF_CUDA(cudaSetDevice(h->device), h->err);
  const cudaIpcMemHandle_t* in = reinterpret_cast<const cudaIpcMemHandle_t*>(handles);
  for (int i = 0; i < 8; ++i)
    PF_CUDA(cudaIpcOpenMemHandle(&h->peer[peer][i], in[i], cudaIpcMemLazyEnablePeerAccess), h->err);
  h->peer_ipc[peer] = true;
  return PF_OK;
}

int pf_shard_exchange(pf_handle* h, void** out4) {
  if (!h || !out4 || h->n_shards < 2) return PF_EINVAL;
  out4[0] = h->tsync;    // uint64 max key (send, 8 B)
  out4[1] = h->sh_gmax;  // uint64 [n_shards] (receive)
  out4[2] = h->sh_send;  // int64 [4] (send)
  out4[3] = h->sh_gsum;  // int64 [n_shards][4] (receive)
  return PF_OK;
}

void* pf_shard_stream(pf_handle* h) { return h ? (void*)h->stream : nullptr; }

int pf_shard_begin(pf_handle* h, const uint8_t* frames, int32_t F, int32_t on_device) {
  if (!h || !frames || F < 1 || h->n_shards < 2) return PF_EINVAL;
  PF_CUDA(cudaSetDevice(h->device), h->err);
  h->launches = 0;
  const size_t fbytes = (size_t)F * h->H * h->W;
  const size_t map_elems = (size_t)h->Hm * h->Wm;
  int rc;
  if ((rc = grow((void**)&h->d_maps, &h->maps_cap, (size_t)F * map_elems * h->rs, h->err))) return rc;
  if ((rc = grow((void**)&h->d_traj, &h->traj_cap, (size_t)F * 2 * 8, h->err))) return rc;
  const uint8_t* dframes = frames;
  if (!on_device) {
    if ((rc = grow((void**)&h->d_frames, &h->frames_cap, fbytes, h->err))) return rc;
    PF_CUDA(cudaMemcpyAsync(h->d_frames, frames, fbytes, cudaMemcpyHostToDevice, h->stream), h->err);
    dframes = h->d_frames;
  }
  PF_CUDA(cudaEventRecord(h->ev[0], h->stream), h->err);
  if ((rc = launch_maps(h, dframes, F))) return rc;
  h->sh_F = F;
  return PF_OK;
}

int pf_shard_fused(pf_handle* h, int32_t f) {
  if (!h || h->n_shards < 2 || f < 0 || f >= h->sh_F) return PF_EINVAL;
  PF_CUDA(cudaSetDevice(h->device), h->err);
  const size_t map_elems = (size_t)h->Hm * h->Wm;
  const char* slot = (const char*)h->d_maps + (size_t)f * map_elems * h->rs;
  return launch_frame(h, slot, (long long)h->sh_F * map_elems, f, h->sh_F);
}

static pfk::ShardArgs shard_args(pf_handle* h, int f) {
  pfk::ShardArgs a{};
  a.K = h->K;
  a.n_tiles = h->n_tiles;
  a.n_local = h->nl;
  a.tile0 = h->tile0;
  a.Q = h->Q;
  a.n_shards = h->n_shards;
  a.shard = h->shard;
  a.n_chunks = h->sh_chunks;
  a.gmax = h->sh_gmax;
  a.gsum = h->sh_gsum;
  a.rec_m = h->rec_m;
  a.rec_S = h->rec_S;
  a.rec_X = h->rec_X;
  a.rec_Y = h->rec_Y;
  a.mass = h->sh_mass;
  a.ctot = h->sh_ctot;
  a.croots = h->sh_croots;
  a.sendsum = h->sh_send;
  a.maxkey = h->tsync;
  a.tab_s = h->tab_s;
  a.tab_O = h->tab_O;
  a.tab_invM = h->tab_invM;
  a.win.n_shards = h->n_shards;
  a.win.shard_tiles = h->shard_tiles;
  for (int sh = 0; sh < h->n_shards; ++sh) a.win.win[sh] = (int2*)h->peer[sh][7];
  a.u_out = h->u;
  const pfr::Affine fu =
      pfr::affine_pow((unsigned long long)h->frame_counter * (2ULL * h->K + 1) + 2ULL * (unsigned long long)h->K);
  a.ua = fu.a;
  a.uc = fu.c;
  a.x0 = h->x0;
  a.traj = h->d_traj;
  a.traj_index = f;
  if (h->n_shards == 1) {  // split table of an unsharded track: no exchange
    a.gmax = h->tsync;
    a.gsum = h->sh_send;
  }
  a.degenerate = h->d_degen;
  a.t = (int)h->frame_counter;
  return a;
}

static int shard_tables_launch(pf_handle* h, int traj_index, int traj_stride) {
  (void)traj_stride;  // one track
  const pfk::ShardArgs a = shard_args(h, traj_index);
  if (h->km == 0) {
    pfk::pf_shard_mass<0><<<h->sh_chunks, pfk::kShardChunk, 0, h->stream>>>(a);
    pfk::pf_shard_sum<0><<<1, 1024, 0, h->stream>>>(a);
    pfk::pf_shard_finish<0><<<h->sh_chunks, pfk::kShardChunk, 0, h->stream>>>(a);
  } else if (h->km == 1) {
    pfk::pf_shard_mass<1><<<h->sh_chunks, pfk::kShardChunk, 0, h->stream>>>(a);
    pfk::pf_shard_sum<1><<<1, 1024, 0, h->stream>>>(a);
    pfk::pf_shard_finish<1><<<h->sh_chunks, pfk::kShardChunk, 0, h->stream>>>(a);
  } else {
    pfk::pf_shard_mass<2><<<h->sh_chunks, pfk::kShardChunk, 0, h->stream>>>(a);
    pfk::pf_shard_sum<2><<<1, 1024, 0, h->stream>>>(a);
    pfk::pf_shard_finish<2><<<h->sh_chunks, pfk::kShardChunk, 0, h->stream>>>(a);
  }
  PF_CUDA(cudaGetLastError(), h->err);
  return PF_OK;
}

int pf_shard_tables(pf_handle* h) {
  if (!h || h->n_shards < 2) return PF_EINVAL;
  PF_CUDA(cudaSetDevice(h->device), h->err);
  const pfk::ShardArgs a = shard_args(h, 0);
  const int km = h->km;
  if (km == 0) {
    pfk::pf_shard_mass<0><<<h->sh_chunks, pfk::kShardChunk, 0, h->stream>>>(a);
    pfk::pf_shard_sum<0><<<1, 1024, 0, h->stream>>>(a);
  } else if (km == 1) {
    pfk::pf_shard_mass<1><<<h->sh_chunks, pfk::kShardChunk, 0, h->stream>>>(a);
    pfk::pf_shard_sum<1><<<1, 1024, 0, h->stream>>>(a);
  } else {
    pfk::pf_shard_mass<2><<<h->sh_chunks, pfk::kShardChunk, 0, h->stream>>>(a);
    pfk::pf_shard_sum<2><<<1, 1024, 0, h->stream>>>(a);
  }
  PF_CUDA(cudaGetLastError(), h->err);
  h->launches += 2;
  return PF_OK;
}

int pf_shard_finish(pf_handle* h, int32_t f) {
  if (!h || h->n_shards < 2 || f < 0 || f >= h->sh_F) return PF_EINVAL;
  PF_CUDA(cudaSetDevice(h->device), h->err);
  const pfk::ShardArgs a = shard_args(h, f);
  if (h->km == 0)
    pfk::pf_shard_finish<0><<<h->sh_chunks, pfk::kShardChunk, 0, h->stream>>>(a);
  else if (h->km == 1)
    pfk::pf_shard_finish<1><<<h->sh_chunks, pfk::kShardChunk, 0, h->stream>>>(a);
  else
    pfk::pf_shard_finish<2><<<h->sh_chunks, pfk::kShardChunk, 0, h->stream>>>(a);
  PF_CUDA(cudaGetLastError(), h->err);
  h->launches += 1;
  h->cur = 1 - h->cur;
  h->frame_counter += 1;
  return PF_OK;
}

int pf_shard_end(pf_handle* h, int32_t F, double* traj_out) {
  if (!h || h->n_shards < 2 || F < 1 || F > h->sh_F || !traj_out) return PF_EINVAL;
  PF_CUDA(cudaSetDevice(h->device), h->err);
  PF_CUDA(cudaEventRecord(h->ev[3], h->stream), h->err);
  PF_CUDA(cudaMemcpyAsync(traj_out, h->d_traj, (size_t)F * 2 * 8, cudaMemcpyDeviceToHost, h->stream), h->err);
  int rc = queue_degenerate(h);
  if (rc) return rc;
  PF_CUDA(cudaEventRecord(h->ev[4], h->stream), h->err);
  PF_CUDA(cudaStreamSynchronize(h->stream), h->err);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, h->ev[0], h->ev[4]);
  h->timings[0] = ms;
  return finish_degenerate(h);
}

int pf_shard_local_allgather(pf_handle* const* hs, int32_t S, int32_t which) {
  if (!hs || S < 2 || S > PF_MAX_SHARDS || which < 0 || which > 2) return PF_EINVAL;
  for (int r = 0; r < S; ++r)
    if (!hs[r] || hs[r]->n_shards != S || hs[r]->shard != r) return PF_EINVAL;
  auto cross_wait = [&]() -> int {
    for (int r = 0; r < S; ++r) {
      PF_CUDA(cudaSetDevice(hs[r]->device), hs[r]->err);
      PF_CUDA(cudaEventRecord(hs[r]->xev, hs[r]->stream), hs[r]->err);
    }
    for (int r = 0; r < S; ++r)
      for (int q = 0; q < S; ++q)
        if (q != r) PF_CUDA(cudaStreamWaitEvent(hs[r]->stream, hs[q]->xev, 0), hs[r]->err);
    return PF_OK;
  };
  int rc = cross_wait();
  if (rc || which == 2) return rc;
  for (int r = 0; r < S; ++r) {
    for (int q = 0; q < S; ++q) {
      void* dst = which == 0 ? (void*)(hs[r]->sh_gmax + q) : (void*)(hs[r]->sh_gsum + 4 * q);
      const void* src = which == 0 ? (const void*)hs[q]->tsync : (const void*)hs[q]->sh_send;
      PF_CUDA(cudaMemcpyAsync(dst, src, which == 0 ? 8 : 32, cudaMemcpyDeviceToDevice, hs[r]->stream), hs[r]->err);
    }
  }
  return cross_wait();  // no source is overwritten before every shard copied it
}

// ---------------------------------------------------------------------------
// systematic_ancestors / RNG helpers
// ---------------------------------------------------------------------------
int pf_systematic_ancestors(const double* cdf, int64_t K, double u, int64_t* anc_out, int32_t device) {
  if (!cdf || !anc_out || K < 1) return PF_EINVAL;
  PF_CUDA(cudaSetDevice(device), g_err);
  double* dc = nullptr;
  long long* da = nullptr;
  PF_CUDA(cudaMalloc(&dc, K * 8), g_err);
  PF_CUDA(cudaMalloc(&da, K * 8), g_err);
  PF_CUDA(cudaMemcpy(dc, cdf, K * 8, cudaMemcpyHostToDevice), g_err);
  pfs::st_systematic<<<(unsigned)((K + 255) / 256), 256>>>(K, dc, u, da);
  PF_CUDA(cudaGetLastError(), g_err);
  PF_CUDA(cudaMemcpy(anc_out, da, K * 8, cudaMemcpyDeviceToHost), g_err);
  cudaFree(dc);
  cudaFree(da);
  return PF_OK;
}

int pf_rng_normals(uint64_t seed, uint64_t pos, int64_t n, double* out, int32_t device) {
  if (!out || n < 0) return PF_EINVAL;
  if (n == 0) return PF_OK;
  PF_CUDA(cudaSetDevice(device), g_err);
  int rc = init_device_tables(device, g_err);
  if (rc) return rc;
  double* d = nullptr;
  PF_CUDA(cudaMalloc(&d, n * 8), g_err);
  pfs::st_rng_normals<<<(unsigned)((n + 255) / 256), 256>>>(pfr::seed_state(seed), pos, n, d);
  PF_CUDA(cudaGetLastError(), g_err);
  PF_CUDA(cudaMemcpy(out, d, n * 8, cudaMemcpyDeviceToHost), g_err);
  cudaFree(d);
  return PF_OK;
}

int pf_rng_uniforms(uint64_t seed, uint64_t pos, int64_t n, double* out, int32_t device) {
  if (!out || n < 0) return PF_EINVAL;
  if (n == 0) return PF_OK;
  PF_CUDA(cudaSetDevice(device), g_err);
  int rc = init_device_tables(device, g_err);
  if (rc) return rc;
  double* d = nullptr;
  PF_CUDA(cudaMalloc(&d, n * 8), g_err);
  pfs::st_rng_uniforms<<<(unsigned)((n + 255) / 256), 256>>>(pfr::seed_state(seed), pos, n, d);
  PF_CUDA(cudaGetLastError(), g_err);
  PF_CUDA(cudaMemcpy(out, d, n * 8, cudaMemcpyDeviceToHost), g_err);
  cudaFree(d);
  return PF_OK;
}

}  // extern "C"

#include "pf_stage_api.inc"

// ---------------------------------------------------------------------------
// NumPy-compatible reference stream on the device (staged parity engine)
// ---------------------------------------------------------------------------
struct pf_philox {
  PhxGen g;
  double* buf = nullptr;
  long long cap = 0;
  int device = 0;
};

extern "C" {

int pf_philox_create(pf_philox** out, const uint64_t* state11, int32_t device) {
  if (!out || !state11) return PF_EINVAL;
  *out = nullptr;
  PF_CUDA(cudaSetDevice(device), g_err);
  int rc = init_device_tables(device, g_err);
  if (rc) return rc;
  pf_philox* p = new pf_philox();
  p->device = device;
  if ((rc = p->g.init(state11, g_err))) {
    p->g.release();
    delete p;
    return rc;
  }
  *out = p;
  return PF_OK;
}

int pf_philox_destroy(pf_philox* p) {
  if (!p) return PF_OK;
  cudaSetDevice(p->device);
  p->g.release();
  if (p->buf) cudaFree(p->buf);
  delete p;
  return PF_OK;
}

static int philox_draw(pf_philox* p, int64_t n, double* out, bool normals) {
  if (!p || !out || n < 0) return PF_EINVAL;
  if (n == 0) return PF_OK;
  PF_CUDA(cudaSetDevice(p->device), g_err);
  if (p->cap < n) {
    if (p->buf) cudaFree(p->buf);
    p->buf = nullptr;
    PF_CUDA(cudaMalloc(&p->buf, n * 8), g_err);
    p->cap = n;
  }
  int rc = normals ? p->g.draw(nullptr, n, p->buf, nullptr, g_err) : p->g.uniforms(nullptr, n, p->buf, g_err);
  if (rc) return rc;
  PF_CUDA(cudaMemcpy(out, p->buf, n * 8, cudaMemcpyDeviceToHost), g_err);
  return p->g.check(g_err);
}
int pf_philox_normals(pf_philox* p, int64_t n, double* out) { return philox_draw(p, n, out, true); }
int pf_philox_normals_device(pf_philox* p, int64_t n, double* out_dev, void* stream) {
  if (!p || !out_dev || n < 0) return PF_EINVAL;
  if (n == 0) return PF_OK;
  PF_CUDA(cudaSetDevice(p->device), g_err);
  return p->g.draw((cudaStream_t)stream, n, out_dev, nullptr, g_err);
}
int pf_philox_uniforms(pf_philox* p, int64_t n, double* out) { return philox_draw(p, n, out, false); }

}  // extern "C"
