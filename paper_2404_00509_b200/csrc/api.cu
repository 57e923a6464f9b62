// C ABI of libessl (include/essl.h): context, staging, launch plumbing.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <functional>
#include <memory>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "essl.h"
#include "essl_common.cuh"

namespace essl {
void init_device_decode();
void init_device_pixels();
}

namespace {

thread_local std::string g_err;

int fail(int code, const std::string &msg) {
  g_err = msg;
  return code;
}

#define CK(call)                                                                   \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess)                                                         \
      return fail(ESSL_E_CUDA, std::string(#call ": ") + cudaGetErrorString(e_)); \
  } while (0)

constexpr int kDescRing = 8;

// Context option defaults (essl_option_default reports them).
constexpr int kDefMode = ESSL_DECODE_SPECULATIVE;
constexpr int kDefSeqBits = 3072;
constexpr int kDefCkBits = 64;
constexpr int kDefWarmBits = 2560;  // (2048: -1.4% at 300 steps after the staged list stores)
constexpr int kDefStageBytes = 64 * 1024;
constexpr int kDefGatherCtas = 8;  // (with 4 KB stages; 4 CTAs: 20-step e2e -3%)
constexpr bool kDefGatherTma = true;
constexpr int kDefResizeCols = 2;
constexpr int kDefResizeBand = 64;
constexpr int kDefEarlyExit = 1;

// Persistent host workers for payload staging (one pool per context): a
// batch's copies are split into contiguous ranges, the caller thread takes
// one range and waits for the rest.
class StagePool {
 public:
  explicit StagePool(int n) {
    for (int i = 0; i < n; i++) th_.emplace_back([this, i] { loop(i); });
  }
  ~StagePool() {
    {
      std::lock_guard<std::mutex> g(m_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto &t : th_) t.join();
  }
  int size() const { return (int)th_.size(); }
  // Runs fn(part, nparts) for part in [0, nparts): parts 1.. on the pool, part 0 here.
  void run(int nparts, const std::function<void(int, int)> &fn) {
    nparts = std::max(1, std::min(nparts, (int)th_.size() + 1));
    {
      std::lock_guard<std::mutex> g(m_);
      fn_ = &fn;
      parts_ = nparts;
      pending_ = nparts - 1;
      gen_++;
    }
    cv_.notify_all();
    fn(0, nparts);
    std::unique_lock<std::mutex> l(m_);
    done_.wait(l, [this] { return pending_ == 0; });
    fn_ = nullptr;
  }

 private:
  void loop(int i) {
    uint64_t seen = 0;
    while (true) {
      const std::function<void(int, int)> *fn;
      int parts;
      {
        std::unique_lock<std::mutex> l(m_);
        cv_.wait(l, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
        fn = fn_;
        parts = parts_;
      }
      if (i + 1 < parts) {
        (*fn)(i + 1, parts);
        std::lock_guard<std::mutex> g(m_);
        if (--pending_ == 0) done_.notify_one();
      }
    }
  }
  std::vector<std::thread> th_;
  std::mutex m_;
  std::condition_variable cv_, done_;
  const std::function<void(int, int)> *fn_ = nullptr;
  int parts_ = 0, pending_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

}  // namespace

struct essl_dataset {  // record table of a container (essl_batch_enqueue)
  std::vector<uint64_t> offset;
  std::vector<uint32_t> length, crc;
  std::vector<uint16_t> width, height;
  std::vector<int64_t> label;
};

struct essl_ctx {
  int device = 0;
  int max_batch = 0, max_side = 0, max_payload = 0;
  essl::Scratch s{};
  // descriptor ring (pinned host -> device)
  essl_sample *h_desc[kDescRing] = {};
  essl_sample *d_desc[kDescRing] = {};
  cudaEvent_t ev_desc[kDescRing] = {};
  cudaEvent_t ev_wait = nullptr;  // essl_batch_enqueue's wait on the consumer stream
  bool desc_used[kDescRing] = {};
  int desc_next = 0;
  int64_t *h_il[kDescRing] = {};    // essl_batch_enqueue: indices + labels, same ring slots
  essl_aug *h_aug[kDescRing] = {};  // 3-Aug parameters, same ring slots
  essl_aug *d_aug[kDescRing] = {};
  // 3-Aug scratch: resized uint8 images and their blurred copies (grown on demand)
  uint8_t *aug_a = nullptr, *aug_b = nullptr;
  uint64_t aug_cap = 0;
  // staging (pinned ring, two slots)
  uint8_t *h_stage[2] = {};
  uint8_t *d_stage[2] = {};
  uint64_t stage_cap = 0;
  cudaEvent_t ev_stage[2] = {};
  bool stage_used[2] = {};
  std::unique_ptr<StagePool> stage_pool;  // created on first staged batch
  essl::GatherDesc *h_gather[2] = {}, *d_gather[2] = {};  // pinned-container gathers
  // misc device buffers
  uint64_t *d_offsets = nullptr;  // crop / dump output offsets
  int mode = kDefMode;
  int seq_bits = kDefSeqBits;
  int ck_bits = kDefCkBits;  // (ESSL_OPT_CHECKPOINT_BITS: kept for the API, no effect)
  int warm_bits = kDefWarmBits;
  int stage_max = kDefStageBytes;
  int gather_ctas = kDefGatherCtas;  // k_host_gather grid (ESSL_OPT_GATHER_CTAS)
  bool gather_tma = kDefGatherTma;   // ESSL_OPT_GATHER_TMA: bulk (TMA) bus reads, e2e +9% over LSU loads
  int resize_cols = kDefResizeCols;  // ESSL_OPT_RESIZE_COLS
  int resize_band = kDefResizeBand;  // ESSL_OPT_RESIZE_BAND
  int early_exit = kDefEarlyExit;    // ESSL_OPT_EARLY_EXIT
  int32_t *dbg_lanes = nullptr;  // ESSL_OPT_DEBUG_LANES buffer
  essl::CtaTrace trace{nullptr, nullptr, 0};  // ESSL_OPT_TRACE  // bulk-copy (TMA) gather (ESSL_OPT_GATHER_TMA)
  std::atomic<int64_t> launches{0};
  // profiling: event pairs per launch
  bool profile = false;
  uint32_t profile_mask = 0xFFFFFFFFu;  // ESSL_OPT_PROFILE_KERNELS: which launches are bracketed
  struct Rec { int kid; cudaEvent_t a, b; };
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> pool;
  cudaEvent_t take() {
    if (!pool.empty()) { cudaEvent_t e = pool.back(); pool.pop_back(); return e; }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
};

namespace {
// NVTX range over a host-side stage (header-only NVTX3: a no-op unless a
// profiler is attached), visible in Nsight Systems next to the kernels.
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

// Makes the context's device current for the duration of an entry point and
// restores the caller's device (a context may live on a non-current device).
struct DevGuard {
  int prev = -1;
  explicit DevGuard(const essl_ctx *c) : DevGuard(c ? c->device : -1) {}
  explicit DevGuard(int device) {
    if (device < 0) return;
    int cur = 0;
    if (cudaGetDevice(&cur) == cudaSuccess && cur != device && cudaSetDevice(device) == cudaSuccess)
      prev = cur;
  }
  ~DevGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// Bracket a launch with events when profiling (ESSL_OPT_PROFILE).
struct Prof {
  essl_ctx *c; int kid; cudaStream_t st; cudaEvent_t a = nullptr;
  bool on;
  Prof(essl_ctx *c_, int k, cudaStream_t s)
      : c(c_), kid(k), st(s), on(c_ && c_->profile && ((c_->profile_mask >> k) & 1u)) {
    if (on) { a = c->take(); cudaEventRecord(a, st); }
  }
  ~Prof() {
    if (c) c->launches += 1;
    if (on) {
      cudaEvent_t b = c->take();
      cudaEventRecord(b, st);
      c->recs.push_back({kid, a, b});
    }
  }
};
}  // namespace

namespace {

// Next descriptor ring slot, once the batch that last used it has completed
// (its ev_desc was recorded after that batch's last kernel).
int pick_slot(essl_ctx *c) {
  const int r = c->desc_next;
  c->desc_next = (c->desc_next + 1) % kDescRing;
  if (c->desc_used[r]) CK(cudaEventSynchronize(c->ev_desc[r]));
  c->desc_used[r] = true;
  return r;
}

int pick_desc(essl_ctx *c, const essl_sample *samples, int n, cudaStream_t st,
              essl_sample **d_out) {
  const int r = pick_slot(c);
  if (r < 0) return r;
  std::memcpy(c->h_desc[r], samples, sizeof(essl_sample) * n);
  CK(cudaMemcpyAsync(c->d_desc[r], c->h_desc[r], sizeof(essl_sample) * n,
                     cudaMemcpyHostToDevice, st));
  *d_out = c->d_desc[r];
  return r;
}

// Validate a host essl_aug array; *max_radius = largest blur radius (0: none).
int check_aug(const essl_aug *aug, int n, int *max_radius, bool *any) {
  *max_radius = 0;
  *any = false;
  for (int i = 0; i < n; i++) {
    const essl_aug &a = aug[i];
    if (a.op < ESSL_AUG_OP_NONE || a.op > ESSL_AUG_OP_BLUR || (a.jitter != 0 && a.jitter != 1))
      return fail(ESSL_E_ARG, "essl_aug: bad op / jitter");
    if (a.op == ESSL_AUG_OP_BLUR) {
      if (a.radius < 1 || a.radius > ESSL_AUG_MAX_RADIUS)
        return fail(ESSL_E_ARG, "essl_aug: blur radius out of [1, ESSL_AUG_MAX_RADIUS]");
      *max_radius = std::max(*max_radius, a.radius);
    }
    *any = *any || a.op != ESSL_AUG_OP_NONE || a.jitter;
  }
  return ESSL_OK;
}

// Grow the 3-Aug scratch to `bytes` per buffer (cudaFree synchronises the
// device, so no in-flight batch still reads the old buffers).
int ensure_aug_scratch(essl_ctx *c, uint64_t bytes) {
  if (bytes <= c->aug_cap) return ESSL_OK;
  if (c->aug_a) CK(cudaFree(c->aug_a));
  if (c->aug_b) CK(cudaFree(c->aug_b));
  c->aug_a = c->aug_b = nullptr;
  c->aug_cap = 0;
  CK(cudaMalloc(&c->aug_a, bytes));
  CK(cudaMalloc(&c->aug_b, bytes));
  c->aug_cap = bytes;
  return ESSL_OK;
}

// All of a batch's host->device copies are issued before its kernels: a copy
// queued behind this batch's kernels would hold up the copies (and so the
// kernels) of batches on other streams on the shared copy engine.
int launch_decode(essl_ctx *c, const uint8_t *blob, const essl_sample *d_desc, int n, int max_len,
                  essl_result *results, cudaStream_t st);
int rrc_impl(essl_ctx *c, const uint8_t *blob, const essl_sample *samples, int slot,
             const essl_aug *aug, int n, int res, int out_kind, void *out, int64_t out_stride,
             uint8_t *out_u8, int patch, const int64_t *ids_restore, int n_keep,
             void *tokens_bf16, essl_result *results, cudaStream_t st);

// Pinned-container gather of a batch: samples[i].offset holds the payload's
// container offset on entry and its offset inside the staging slot on return.
int stage_pinned_impl(essl_ctx *c, int slot, const uint8_t *dev_base, essl_sample *samples, int n,
                      cudaStream_t st, const uint8_t **dev_blob, int chain_ctas) {
  if (c->stage_used[slot]) CK(cudaEventSynchronize(c->ev_stage[slot]));
  essl::GatherDesc *h = c->h_gather[slot];
  uint64_t pos = 0;
  for (int i = 0; i < n; i++) {
    const uint32_t len = samples[i].length;
    if ((int)len > c->max_payload) return fail(ESSL_E_CAPACITY, "payload larger than max_payload");
    h[i].src = samples[i].offset;
    h[i].dst = pos;
    h[i].len = len;
    samples[i].offset = pos;
    pos += ((uint64_t)len + 63) / 64 * 64;
  }
  if (n > 0) {
    CK(cudaMemcpyAsync(c->d_gather[slot], h, sizeof(essl::GatherDesc) * n, cudaMemcpyHostToDevice, st));
    // chained gathers (a pipeline fill) run one after the other across every
    // context of the device, each on more CTAs: the oldest batch's payloads
    // arrive first instead of all batches' together
    static std::mutex chain_m;
    static std::vector<cudaEvent_t> chain_tail;
    std::unique_lock<std::mutex> lk(chain_m, std::defer_lock);
    if (chain_ctas > 0) {
      lk.lock();
      if ((int)chain_tail.size() <= c->device) chain_tail.resize(c->device + 1, nullptr);
      if (!chain_tail[c->device]) CK(cudaEventCreateWithFlags(&chain_tail[c->device], cudaEventDisableTiming));
      else CK(cudaStreamWaitEvent(st, chain_tail[c->device], 0));
    }
    {
      Prof pr(c, ESSL_K_STAGE, st);
      essl::launch_host_gather(dev_base, c->d_gather[slot], n, c->d_stage[slot],
                               chain_ctas > 0 ? chain_ctas : c->gather_ctas, c->gather_tma, st);
    }
    if (chain_ctas > 0) CK(cudaEventRecord(chain_tail[c->device], st));
  }
  CK(cudaEventRecord(c->ev_stage[slot], st));
  c->stage_used[slot] = true;
  *dev_blob = c->d_stage[slot];
  return ESSL_OK;
}

int run_decode(essl_ctx *c, const uint8_t *blob, const essl_sample *samples, int n,
               essl_result *results, cudaStream_t st, int *ring, const essl_aug *aug = nullptr) {
  if (n > c->max_batch) return fail(ESSL_E_CAPACITY, "batch larger than context max_batch");
  int max_len = 0;
  for (int i = 0; i < n; i++) {
    if ((int)samples[i].length > c->max_payload)
      return fail(ESSL_E_CAPACITY, "payload larger than context max_payload");
    max_len = std::max(max_len, (int)samples[i].length);
  }
  essl_sample *d_desc = nullptr;
  int r = pick_desc(c, samples, n, st, &d_desc);
  if (r < 0) return r;
  *ring = r;
  if (aug) {
    std::memcpy(c->h_aug[r], aug, sizeof(essl_aug) * n);
    CK(cudaMemcpyAsync(c->d_aug[r], c->h_aug[r], sizeof(essl_aug) * n, cudaMemcpyHostToDevice, st));
  }
  return launch_decode(c, blob, d_desc, n, max_len, results, st);
}

// k_prep -> k_entropy -> k_idct of a batch whose descriptors are on the device.
int launch_decode(essl_ctx *c, const uint8_t *blob, const essl_sample *d_desc, int n, int max_len,
                  essl_result *results, cudaStream_t st) {
  CK(cudaMemsetAsync(c->s.counters, 0, 4 * sizeof(unsigned long long), st));
  essl::DecodeParams p;
  p.blob = blob;
  p.samples = d_desc;
  p.n = n;
  p.s = c->s;
  p.mode = c->mode;
  p.seq_bits = c->seq_bits;
  p.warm_bits = c->warm_bits;
  p.stage_bytes = c->stage_max;
  p.early_exit = c->early_exit;
  p.results = results;
  p.dbg_lanes = c->dbg_lanes;
  p.trace = c->trace;
  {
    Prof pr(c, ESSL_K_PREP, st);
    essl::launch_prep(p, st, max_len);
  }
  {
    Prof pr(c, ESSL_K_ENTROPY, st);
    essl::launch_entropy(p, st, max_len);
  }
  {
    Prof pr(c, ESSL_K_IDCT, st);
    essl::launch_idct(p, st);
  }
  CK(cudaGetLastError());
  return ESSL_OK;
}

}  // namespace

extern "C" {

const char *essl_last_error(void) { return g_err.c_str(); }
const char *essl_version(void) { return "essl-b200 0.1 (sm_100a)"; }

int essl_memcpy_async(void *dst, const void *src, uint64_t bytes, void *stream) {
  if (bytes && (!dst || !src)) return fail(ESSL_E_ARG, "essl_memcpy_async: null pointer");
  if (!bytes) return ESSL_OK;
  CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, (cudaStream_t)stream));
  return ESSL_OK;
}

int essl_ctx_create(int device, int max_batch, int max_side, int max_payload, int flags,
                    essl_ctx **out) {
  (void)flags;
  if (!out || max_batch < 1 || max_side < 1 || max_payload < 4 || max_payload > (1 << 22))
    return fail(ESSL_E_ARG, "essl_ctx_create: bad arguments");
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(ESSL_E_ARG, "essl_ctx_create: no such device");
  DevGuard dg_(device);  // the caller's current device is restored on return
  essl_ctx *c = new essl_ctx();
  c->device = device;
  c->max_batch = max_batch;
  c->max_side = max_side;
  c->max_payload = max_payload;
  // worst-case per-image scratch (4:4:4 / h,v<=4 padding included)
  const uint64_t side_blocks = (uint64_t)(max_side + 7) / 8 + 4;
  const uint64_t blocks = 3 * side_blocks * side_blocks;
  const uint64_t mcus = ((uint64_t)max_side + 7) / 8 * (((uint64_t)max_side + 7) / 8);
  c->s.clean_cap = (uint64_t)max_batch * (((uint64_t)max_payload + 128 + 4 * (mcus + 2) + 64 + 15) / 16 * 16);
  c->s.coef_cap = (uint64_t)max_batch * blocks * 64;
  c->s.plane_cap = (uint64_t)max_batch * blocks * 64 + 16 * (uint64_t)max_batch;
  auto cleanup = [&](int code) {
    essl_ctx_destroy(c);
    return code;
  };
#define CKC(call)                                                                   \
  do {                                                                              \
    cudaError_t e_ = (call);                                                        \
    if (e_ != cudaSuccess)                                                          \
      return cleanup(fail(ESSL_E_CUDA, std::string(#call ": ") + cudaGetErrorString(e_))); \
  } while (0)
  CKC(cudaMalloc(&c->s.clean, c->s.clean_cap));
  CKC(cudaMalloc(&c->s.coef, c->s.coef_cap * sizeof(int16_t)));
  CKC(cudaMalloc(&c->s.plane, c->s.plane_cap));
  CKC(cudaMalloc(&c->s.counters, 4 * sizeof(unsigned long long)));
  CKC(cudaMalloc(&c->s.info, sizeof(essl::ImgInfo) * max_batch));
  CKC(cudaMalloc(&c->s.hdr, essl::decode_hdr_bytes() * max_batch));
  CKC(cudaMalloc(&c->s.tabcache, essl::tabcache_bytes()));
  CKC(cudaMemset(c->s.tabcache, 0, essl::tabcache_bytes()));
  // unit lists + block records per image: lanes x (cap + 24 + 2 (cap/2 + 26)
  // + 3) u32 (k_entropy's stride), cap = (slen + warm + continuation)/4 + 68,
  // lanes x slen <= 8 x payload
  c->s.list_cap = (uint64_t)max_batch *
                  (4ull * max_payload + (uint64_t)essl::kEntropyLanes *
                                            (2ull * ((essl::kMaxWarmBits + essl::kContinuationBits) / 4 + 68) + 80) + 8);
  // (+ 4 words per entropy lane past the pool: slack for the bounds checks)
  CKC(cudaMalloc(&c->s.list, (c->s.list_cap + 4 * essl::kEntropyLanes) * sizeof(uint32_t)));
  CKC(cudaMalloc(&c->d_offsets, sizeof(uint64_t) * max_batch));
  for (int r = 0; r < kDescRing; r++) {
    CKC(cudaMallocHost(&c->h_desc[r], sizeof(essl_sample) * max_batch));
    CKC(cudaMalloc(&c->d_desc[r], sizeof(essl_sample) * max_batch));
    CKC(cudaEventCreateWithFlags(&c->ev_desc[r], cudaEventDisableTiming));
    CKC(cudaMallocHost(&c->h_aug[r], sizeof(essl_aug) * max_batch));
    CKC(cudaMallocHost(&c->h_il[r], 2 * sizeof(int64_t) * max_batch));
    CKC(cudaMalloc(&c->d_aug[r], sizeof(essl_aug) * max_batch));
  }
  CKC(cudaEventCreateWithFlags(&c->ev_wait, cudaEventDisableTiming));
  c->stage_cap = (uint64_t)max_batch * (((uint64_t)max_payload + 63) / 64 * 64);
  for (int r = 0; r < 2; r++) {
    CKC(cudaMallocHost(&c->h_stage[r], c->stage_cap));
    CKC(cudaMalloc(&c->d_stage[r], c->stage_cap));
    CKC(cudaEventCreateWithFlags(&c->ev_stage[r], cudaEventDisableTiming));
    CKC(cudaMallocHost(&c->h_gather[r], sizeof(essl::GatherDesc) * max_batch));
    CKC(cudaMalloc(&c->d_gather[r], sizeof(essl::GatherDesc) * max_batch));
  }
  // per-device state (CRC tables, normalize LUTs, shared-memory opt-ins) is
  // set up once for every device a context lives on
  {
    static std::mutex m;
    static std::vector<bool> done;
    std::lock_guard<std::mutex> g(m);
    if ((int)done.size() <= device) done.resize(device + 1, false);
    if (!done[device]) {
      essl::init_device_decode();
      essl::init_device_pixels();
      CKC(cudaDeviceSynchronize());  // tables ready before any stream's first batch
      done[device] = true;
    }
  }
#undef CKC
  *out = c;
  return ESSL_OK;
}

int essl_ctx_destroy(essl_ctx *c) {
  if (!c) return ESSL_OK;
  DevGuard dg_(c);
  cudaDeviceSynchronize();
  cudaFree(c->s.clean);
  cudaFree(c->s.coef);
  cudaFree(c->s.plane);
  cudaFree(c->s.counters);
  cudaFree(c->s.info);
  cudaFree(c->s.hdr);
  if (c->ev_wait) cudaEventDestroy(c->ev_wait);
  cudaFree(c->s.tabcache);
  cudaFree(c->s.list);
  cudaFree(c->d_offsets);
  for (int r = 0; r < kDescRing; r++) {
    if (c->h_desc[r]) cudaFreeHost(c->h_desc[r]);
    if (c->d_desc[r]) cudaFree(c->d_desc[r]);
    if (c->ev_desc[r]) cudaEventDestroy(c->ev_desc[r]);
    if (c->h_aug[r]) cudaFreeHost(c->h_aug[r]);
    if (c->h_il[r]) cudaFreeHost(c->h_il[r]);
    if (c->d_aug[r]) cudaFree(c->d_aug[r]);
  }
  if (c->dbg_lanes) cudaFree(c->dbg_lanes);
  if (c->trace.buf) { cudaFree(c->trace.buf); cudaFree(c->trace.count); }
  if (c->aug_a) cudaFree(c->aug_a);
  if (c->aug_b) cudaFree(c->aug_b);
  for (int r = 0; r < 2; r++) {
    if (c->h_stage[r]) cudaFreeHost(c->h_stage[r]);
    if (c->d_stage[r]) cudaFree(c->d_stage[r]);
    if (c->ev_stage[r]) cudaEventDestroy(c->ev_stage[r]);
    if (c->h_gather[r]) cudaFreeHost(c->h_gather[r]);
    if (c->d_gather[r]) cudaFree(c->d_gather[r]);
  }
  for (auto &r : c->recs) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
  for (auto e : c->pool) cudaEventDestroy(e);
  delete c;
  return ESSL_OK;
}

int essl_ctx_set_option(essl_ctx *c, int option, int64_t value) {
  if (!c) return fail(ESSL_E_ARG, "null context");
  DevGuard dg_(c);
  switch (option) {
    case ESSL_OPT_DECODE_MODE:
      if (value != ESSL_DECODE_SPECULATIVE && value != ESSL_DECODE_SERIAL)
        return fail(ESSL_E_ARG, "bad decode mode");
      c->mode = (int)value;
      return ESSL_OK;
    case ESSL_OPT_SEQ_BITS:
      if (value < 32 || value > (1 << 24)) return fail(ESSL_E_ARG, "bad seq bits");
      c->seq_bits = (int)value;
      return ESSL_OK;
    case ESSL_OPT_WARMUP_BITS:
      if (value < 0 || value > essl::kMaxWarmBits) return fail(ESSL_E_ARG, "bad warm-up bits");
      c->warm_bits = (int)value;
      return ESSL_OK;
    case ESSL_OPT_STAGE_BYTES:
      if (value < 0 || value > (1 << 20)) return fail(ESSL_E_ARG, "bad stage bytes");
      c->stage_max = (int)value;
      return ESSL_OK;
    case ESSL_OPT_GATHER_CTAS:
      if (value < 0 || value > 65535) return fail(ESSL_E_ARG, "bad gather CTA count");
      c->gather_ctas = (int)value;
      return ESSL_OK;
    case ESSL_OPT_TRACE:
      if (c->trace.buf) {
        CK(cudaFree(c->trace.buf));
        CK(cudaFree(c->trace.count));
        c->trace = essl::CtaTrace{nullptr, nullptr, 0};
      }
      if (value > 0) {
        if (value > (1 << 24)) return fail(ESSL_E_ARG, "trace capacity too large");
        CK(cudaMalloc(&c->trace.buf, sizeof(unsigned long long) * 4 * (size_t)value));
        CK(cudaMalloc(&c->trace.count, sizeof(unsigned int)));
        CK(cudaMemset(c->trace.count, 0, sizeof(unsigned int)));
        c->trace.cap = (unsigned int)value;
      }
      return ESSL_OK;
    case ESSL_OPT_DEBUG_LANES:
      if (value && !c->dbg_lanes) {
        CK(cudaMalloc(&c->dbg_lanes, sizeof(int32_t) * 8 * essl::kEntropyLanes * c->max_batch));
        CK(cudaMemset(c->dbg_lanes, 0xFF, sizeof(int32_t) * 8 * essl::kEntropyLanes * c->max_batch));
      } else if (!value && c->dbg_lanes) {
        CK(cudaFree(c->dbg_lanes));
        c->dbg_lanes = nullptr;
      }
      return ESSL_OK;
    case ESSL_OPT_GATHER_TMA:
      c->gather_tma = value != 0;
      return ESSL_OK;
    case ESSL_OPT_PROFILE:
      c->profile = value != 0;
      return ESSL_OK;
    case ESSL_OPT_RESIZE_COLS:
      if (value != 2 && value != 4 && value != 8) return fail(ESSL_E_ARG, "resize columns must be 2, 4 or 8");
      c->resize_cols = (int)value;
      return ESSL_OK;
    case ESSL_OPT_RESIZE_BAND:
      if (value < 1 || value > essl::kMaxBandRows) return fail(ESSL_E_ARG, "bad resize band");
      c->resize_band = (int)value;
      return ESSL_OK;
    case ESSL_OPT_EARLY_EXIT:
      c->early_exit = value != 0;
      return ESSL_OK;
    case ESSL_OPT_PROFILE_KERNELS:
      c->profile_mask = (uint32_t)value;
      return ESSL_OK;
    case ESSL_OPT_CHECKPOINT_BITS:
      if (value < 1 || value > (1 << 24)) return fail(ESSL_E_ARG, "bad checkpoint bits");
      c->ck_bits = (int)value;
      return ESSL_OK;
  }
  return fail(ESSL_E_ARG, "unknown option");
}

int essl_check_read(uint32_t *out, int n, int reset) {
  if (!out || n < 1) return fail(ESSL_E_ARG, "essl_check_read: bad arguments");
  unsigned int d[essl::CK_COUNT], p[essl::CK_COUNT];
  essl::check_read_decode(d, reset != 0);
  essl::check_read_pixels(p, reset != 0);
  for (int i = 0; i < n && i < essl::CK_COUNT; i++) out[i] = d[i] + p[i];
  CK(cudaGetLastError());
#ifdef ESSL_CHECKED
  return 1;
#else
  return 0;
#endif
}

int essl_abi_sizes(int64_t *out, int n) {
  const int64_t sz[5] = {(int64_t)sizeof(essl_sample), (int64_t)sizeof(essl_result), (int64_t)sizeof(essl_aug),
                         (int64_t)sizeof(essl_batch_cfg), (int64_t)sizeof(essl_batch_io)};
  for (int i = 0; i < n && i < 5; i++) out[i] = sz[i];
  return 5;
}

int essl_option_default(int option, int64_t *value) {
  if (!value) return fail(ESSL_E_ARG, "essl_option_default: null value");
  switch (option) {
    case ESSL_OPT_DECODE_MODE: *value = kDefMode; return ESSL_OK;
    case ESSL_OPT_SEQ_BITS: *value = kDefSeqBits; return ESSL_OK;
    case ESSL_OPT_CHECKPOINT_BITS: *value = kDefCkBits; return ESSL_OK;
    case ESSL_OPT_PROFILE: *value = 0; return ESSL_OK;
    case ESSL_OPT_WARMUP_BITS: *value = kDefWarmBits; return ESSL_OK;
    case ESSL_OPT_STAGE_BYTES: *value = kDefStageBytes; return ESSL_OK;
    case ESSL_OPT_GATHER_CTAS: *value = kDefGatherCtas; return ESSL_OK;
    case ESSL_OPT_GATHER_TMA: *value = kDefGatherTma ? 1 : 0; return ESSL_OK;
    case ESSL_OPT_DEBUG_LANES: *value = 0; return ESSL_OK;
    case ESSL_OPT_TRACE: *value = 0; return ESSL_OK;
    case ESSL_OPT_RESIZE_COLS: *value = kDefResizeCols; return ESSL_OK;
    case ESSL_OPT_RESIZE_BAND: *value = kDefResizeBand; return ESSL_OK;
    case ESSL_OPT_EARLY_EXIT: *value = kDefEarlyExit; return ESSL_OK;
    case ESSL_OPT_PROFILE_KERNELS: *value = 0xFFFFFFFF; return ESSL_OK;
  }
  return fail(ESSL_E_ARG, "unknown option");
}

int64_t essl_ctx_launch_count(const essl_ctx *c) { return c ? c->launches.load() : -1; }

int essl_debug_stats(essl_ctx *c, int64_t *out, int n) {
  if (!c || !out || n < 0 || n > c->max_batch) return fail(ESSL_E_ARG, "essl_debug_stats: bad arguments");
  DevGuard dg_(c);
  std::vector<essl::ImgInfo> info(n);
  CK(cudaMemcpy(info.data(), c->s.info, sizeof(essl::ImgInfo) * n, cudaMemcpyDeviceToHost));
  for (int i = 0; i < n; i++) std::memcpy(out + 16 * i, info[i].dbg, 16 * sizeof(int64_t));
  return ESSL_OK;
}

int essl_trace_read(essl_ctx *c, uint64_t *out, int max) {
  if (!c || !out || max < 0 || !c->trace.buf) return fail(ESSL_E_ARG, "essl_trace_read: tracing off");
  DevGuard dg_(c);
  CK(cudaDeviceSynchronize());
  unsigned int n = 0;
  CK(cudaMemcpy(&n, c->trace.count, sizeof(n), cudaMemcpyDeviceToHost));
  n = std::min(n, c->trace.cap);
  n = std::min(n, (unsigned int)max);
  CK(cudaMemcpy(out, c->trace.buf, sizeof(uint64_t) * 4 * n, cudaMemcpyDeviceToHost));
  CK(cudaMemset(c->trace.count, 0, sizeof(unsigned int)));
  return (int)n;
}

int essl_debug_lanes(essl_ctx *c, int32_t *out, int n) {
  if (!c || !out || n < 0 || n > c->max_batch || !c->dbg_lanes)
    return fail(ESSL_E_ARG, "essl_debug_lanes: bad arguments (ESSL_OPT_DEBUG_LANES off?)");
  DevGuard dg_(c);
  CK(cudaMemcpy(out, c->dbg_lanes, sizeof(int32_t) * 8 * essl::kEntropyLanes * n,
                cudaMemcpyDeviceToHost));
  return ESSL_OK;
}

static cudaEvent_t g_mark = nullptr;

int essl_profile_mark(void *stream) {
  if (!g_mark) CK(cudaEventCreate(&g_mark));
  CK(cudaEventRecord(g_mark, (cudaStream_t)stream));
  return ESSL_OK;
}

int essl_ctx_profile_timeline(essl_ctx *c, int32_t *kid, double *t0_ms, double *t1_ms, int max) {
  if (!c || !kid || !t0_ms || !t1_ms || max < 0) return fail(ESSL_E_ARG, "essl_ctx_profile_timeline: bad arguments");
  DevGuard dg_(c);
  if (!g_mark) return fail(ESSL_E_ARG, "essl_profile_mark was not called");
  CK(cudaEventSynchronize(g_mark));
  int n = 0;
  for (auto &r : c->recs) {
    if (n >= max) break;
    CK(cudaEventSynchronize(r.b));
    float a = 0.f, b = 0.f;
    CK(cudaEventElapsedTime(&a, g_mark, r.a));
    CK(cudaEventElapsedTime(&b, g_mark, r.b));
    kid[n] = r.kid;
    t0_ms[n] = a;
    t1_ms[n] = b;
    n++;
  }
  return n;
}

int essl_ctx_profile_read(essl_ctx *c, double *ms, int64_t *count) {
  if (!c || !ms || !count) return fail(ESSL_E_ARG, "essl_ctx_profile_read: bad arguments");
  DevGuard dg_(c);
  for (auto &r : c->recs) {
    CK(cudaEventSynchronize(r.b));
    float t = 0.f;
    CK(cudaEventElapsedTime(&t, r.a, r.b));
    if (r.kid >= 0 && r.kid < ESSL_K_COUNT) {
      ms[r.kid] += t;
      count[r.kid] += 1;
    }
    c->pool.push_back(r.a);
    c->pool.push_back(r.b);
  }
  c->recs.clear();
  return ESSL_OK;
}

int essl_stage(essl_ctx *c, int slot, const uint8_t *const *src, const uint32_t *len, int n,
               essl_sample *samples, int nthreads, void *stream, const uint8_t **dev_blob) {
  if (!c || slot < 0 || slot > 1 || n < 0 || n > c->max_batch || !dev_blob)
    return fail(ESSL_E_ARG, "essl_stage: bad arguments");
  DevGuard dg_(c);
  cudaStream_t st = (cudaStream_t)stream;
  if (c->stage_used[slot]) CK(cudaEventSynchronize(c->ev_stage[slot]));
  std::vector<uint64_t> off(n + 1);
  uint64_t pos = 0;
  for (int i = 0; i < n; i++) {
    if ((int)len[i] > c->max_payload) return fail(ESSL_E_CAPACITY, "payload larger than max_payload");
    off[i] = pos;
    pos += ((uint64_t)len[i] + 63) / 64 * 64;
  }
  off[n] = pos;
  uint8_t *h = c->h_stage[slot];
  nthreads = std::max(1, std::min(nthreads, n));
  if (nthreads > 1 && (!c->stage_pool || c->stage_pool->size() + 1 < nthreads))
    c->stage_pool.reset(new StagePool(nthreads - 1));
  // contiguous ranges of samples with about equal bytes per part
  auto work = [&](int part, int parts) {
    const uint64_t lo = pos * part / parts, hi = pos * (part + 1) / parts;
    int i = (int)(std::upper_bound(off.begin(), off.begin() + n, lo) - off.begin()) - 1;
    for (i = std::max(i, 0); i < n && off[i] < hi; i++)
      if (off[i] >= lo) std::memcpy(h + off[i], src[i], len[i]);
  };
  if (nthreads == 1) work(0, 1);
  else c->stage_pool->run(nthreads, work);
  for (int i = 0; i < n; i++) {
    samples[i].offset = off[i];
    samples[i].length = len[i];
  }
  if (pos) CK(cudaMemcpyAsync(c->d_stage[slot], h, pos, cudaMemcpyHostToDevice, st));
  CK(cudaEventRecord(c->ev_stage[slot], st));
  c->stage_used[slot] = true;
  *dev_blob = c->d_stage[slot];
  return ESSL_OK;
}

int essl_host_register(void *ptr, uint64_t bytes, int readonly) {
  if (!ptr || bytes == 0) return fail(ESSL_E_ARG, "essl_host_register: bad arguments");
  const unsigned flags = cudaHostRegisterPortable | cudaHostRegisterMapped |
                         (readonly ? cudaHostRegisterReadOnly : 0u);
  const cudaError_t e = cudaHostRegister(ptr, bytes, flags);
  if (e != cudaSuccess) {
    (void)cudaGetLastError();  // not sticky: leave no error for later launches
    return fail(ESSL_E_CUDA, std::string("cudaHostRegister: ") + cudaGetErrorString(e));
  }
  return ESSL_OK;
}

int essl_host_unregister(void *ptr) {
  if (!ptr) return fail(ESSL_E_ARG, "essl_host_unregister: null");
  CK(cudaHostUnregister(ptr));
  return ESSL_OK;
}

int essl_host_device_ptr(void *ptr, void **dev_ptr) {
  if (!ptr || !dev_ptr) return fail(ESSL_E_ARG, "essl_host_device_ptr: bad arguments");
  CK(cudaHostGetDevicePointer(dev_ptr, ptr, 0));
  return ESSL_OK;
}

int essl_stage_pinned(essl_ctx *c, int slot, const uint8_t *dev_base, const uint64_t *src_off,
                      const uint32_t *len, int n, essl_sample *samples, void *stream,
                      const uint8_t **dev_blob) {
  if (!c || slot < 0 || slot > 1 || n < 0 || n > c->max_batch || !dev_blob || (n > 0 && (!dev_base || !src_off || !len)))
    return fail(ESSL_E_ARG, "essl_stage_pinned: bad arguments");
  DevGuard dg_(c);
  for (int i = 0; i < n; i++) {
    samples[i].offset = src_off[i];
    samples[i].length = len[i];
  }
  return stage_pinned_impl(c, slot, dev_base, samples, n, (cudaStream_t)stream, dev_blob, 0);
}

int essl_decode_rrc(essl_ctx *c, const uint8_t *blob, const essl_sample *samples, int n, int res,
                    int out_kind, void *out, int64_t out_stride, uint8_t *out_u8,
                    essl_result *results, void *stream) {
  return essl_decode_rrc_aug(c, blob, samples, nullptr, n, res, out_kind, out, out_stride, out_u8,
                             results, stream);
}

int essl_decode_rrc_aug(essl_ctx *c, const uint8_t *blob, const essl_sample *samples,
                        const essl_aug *aug, int n, int res, int out_kind, void *out,
                        int64_t out_stride, uint8_t *out_u8, essl_result *results,
                        void *stream) {
  return essl_decode_rrc_visible(c, blob, samples, aug, n, res, out_kind, out, out_stride, out_u8,
                                 0, nullptr, 0, nullptr, results, stream);
}

int essl_decode_rrc_visible(essl_ctx *c, const uint8_t *blob, const essl_sample *samples,
                            const essl_aug *aug, int n, int res, int out_kind, void *out,
                            int64_t out_stride, uint8_t *out_u8, int patch,
                            const int64_t *ids_restore, int n_keep, void *tokens_bf16,
                            essl_result *results, void *stream) {
  if (!c || n < 0 || res < 1 || (n > 0 && (!blob || !samples)))
    return fail(ESSL_E_ARG, "essl_decode_rrc: bad arguments");
  DevGuard dg_(c);
  return rrc_impl(c, blob, samples, -1, aug, n, res, out_kind, out, out_stride, out_u8, patch,
                  ids_restore, n_keep, tokens_bf16, results, (cudaStream_t)stream);
}

}  // extern "C"

namespace {
// The decode + pixel stage of a batch.  slot < 0: descriptors `samples`
// (host) go through a fresh ring slot; slot >= 0: they are already in that
// slot's pinned buffer (essl_batch_enqueue).
int rrc_impl(essl_ctx *c, const uint8_t *blob, const essl_sample *samples, int slot,
             const essl_aug *aug, int n, int res, int out_kind, void *out, int64_t out_stride,
             uint8_t *out_u8, int patch, const int64_t *ids_restore, int n_keep,
             void *tokens_bf16, essl_result *results, cudaStream_t st) {
  if (out_kind != ESSL_OUT_BF16_NCHW && out_kind != ESSL_OUT_F32_NCHW && out_kind != ESSL_OUT_NONE)
    return fail(ESSL_E_ARG, "bad out_kind");
  if (out_kind != ESSL_OUT_NONE && !out) return fail(ESSL_E_ARG, "null output");
  const bool want_vis = tokens_bf16 != nullptr;
  if (want_vis && (patch < 1 || res % patch || !ids_restore || n_keep < 0 ||
                   n_keep > (res / patch) * (res / patch)))
    return fail(ESSL_E_ARG, "essl_decode_rrc_visible: bad patch / ids_restore / n_keep");
  if (n == 0) return ESSL_OK;
  int max_radius = 0;
  bool any_aug = false;
  if (aug) {
    int rc = check_aug(aug, n, &max_radius, &any_aug);
    if (rc) return rc;
  }
  if (want_vis && any_aug && out_kind != ESSL_OUT_BF16_NCHW)
    return fail(ESSL_E_ARG, "visible tokens with 3-Aug need the bf16 pixel output");
  if (any_aug) {
    int rc = ensure_aug_scratch(c, (uint64_t)n * res * res * 3);
    if (rc) return rc;
  }
  int ring = -1;
  const bool aug_out = any_aug && (out_kind != ESSL_OUT_NONE || out_u8);
  int rc;
  if (slot < 0) {
    rc = run_decode(c, blob, samples, n, results, st, &ring, aug_out ? aug : nullptr);
  } else {
    ring = slot;
    int max_len = 0;
    for (int i = 0; i < n; i++) max_len = std::max(max_len, (int)samples[i].length);
    if (max_len > c->max_payload) return fail(ESSL_E_CAPACITY, "payload larger than context max_payload");
    CK(cudaMemcpyAsync(c->d_desc[slot], c->h_desc[slot], sizeof(essl_sample) * n,
                       cudaMemcpyHostToDevice, st));
    if (aug_out) {
      std::memcpy(c->h_aug[slot], aug, sizeof(essl_aug) * n);
      CK(cudaMemcpyAsync(c->d_aug[slot], c->h_aug[slot], sizeof(essl_aug) * n,
                         cudaMemcpyHostToDevice, st));
    }
    rc = launch_decode(c, blob, c->d_desc[slot], n, max_len, results, st);
  }
  if (rc) return rc;
  essl::PixelParams pp;
  pp.info = c->s.info;
  pp.plane = c->s.plane;
  pp.n = n;
  pp.res = res;
  // 3-Aug: k_resize finishes the point-op images (writing out / out_u8) and
  // leaves blur / jitter images in aug_a for k_aug_blur / k_aug_out
  pp.out_kind = any_aug && !aug_out ? ESSL_OUT_NONE : out_kind;
  pp.out = out;
  pp.out_stride = out_stride;
  pp.out_u8 = any_aug && !aug_out ? c->aug_a : out_u8;
  pp.aug = aug_out ? c->d_aug[ring] : nullptr;
  pp.aug_u8 = c->aug_a;
  // visible tokens fused into k_resize (with 3-Aug they are gathered from
  // the finished pixels after k_aug_out instead)
  pp.vis = want_vis && !any_aug ? tokens_bf16 : nullptr;
  pp.vis_restore = ids_restore;
  pp.patch = want_vis ? patch : 0;
  pp.n_keep = n_keep;
  pp.trace = c->trace;
  {
    // the largest band (output rows per k_resize CTA, <= kMaxBandRows) whose
    // shared staging (source rows x widest crop + the column taps) for this
    // batch's crops stays within 96 KB (two CTAs per SM), else the largest
    // that fits the 200 KB budget; crops wider than that read the planes
    // directly (no staging)
    auto smem = [&](int b) {
      int w = 0;
      for (int i = 0; i < n; i++)
        w = std::max(w, essl::band_source_rows(samples[i].h, res, b) * std::max(samples[i].w, 1));
      pp.band = b;
      pp.src_words = (w + 3) / 4 * 4;
      return essl::resize_smem(pp);
    };
    pp.cols = c->resize_cols;
    // CTAs per SM by registers: 2 (8 columns) / 3 (4) / 4 (2)
    const size_t budget = pp.cols == 8 ? 96 * 1024 : (pp.cols == 4 ? 64 * 1024 : 48 * 1024);
    int band = pp.cols == 2 && !want_vis ? std::min(c->resize_band, 32) : c->resize_band;
    while (band > 8 && smem(band) > budget) band /= 2;
    if (smem(band) > budget) {
      band = c->resize_band;
      while (band > 1 && smem(band) > 200 * 1024) band /= 2;
    }
    if (smem(band) > 200 * 1024) {
      pp.band = c->resize_band;
      pp.src_words = 0;  // unstaged: k_resize reads the planes directly
      if (essl::resize_smem(pp) > 200 * 1024)
        return fail(ESSL_E_CAPACITY, "output resolution too large for the resize kernel");
    }
  }
  if (pp.out_kind != ESSL_OUT_NONE || pp.out_u8 || pp.vis) {
    Prof pr(c, ESSL_K_RESIZE, st);
    essl::launch_resize(pp, st);
  }
  if (aug_out) {
    essl::AugOutParams ap{c->aug_a, c->aug_b, c->d_aug[ring], n, res, res, out_kind, out,
                          out_stride, out_u8, 1};
    Prof pr(c, ESSL_K_AUG, st);
    essl::launch_aug(ap, max_radius, st);
  }
  if (want_vis && any_aug) {
    if (out_stride && out_stride != 3ll * res * res)
      return fail(ESSL_E_ARG, "visible tokens with 3-Aug need dense pixel output");
    Prof pr(c, ESSL_K_GATHER, st);
    essl::launch_gather_restore(out, n, res, patch, ids_restore, n_keep, tokens_bf16, st);
  }
  CK(cudaGetLastError());
  CK(cudaEventRecord(c->ev_desc[ring], st));
  return ESSL_OK;
}
}  // namespace

extern "C" {

int essl_augment_u8(essl_ctx *c, const uint8_t *src, int n, int h, int w, const essl_aug *aug,
                    uint8_t *dst, void *stream) {
  if (!c || n < 0 || h < 1 || w < 1 || (n > 0 && (!src || !dst || !aug)) || src == dst)
    return fail(ESSL_E_ARG, "essl_augment_u8: bad arguments");
  DevGuard dg_(c);
  if (n == 0) return ESSL_OK;
  if (n > c->max_batch) return fail(ESSL_E_CAPACITY, "batch larger than context max_batch");
  if (h > c->max_side || w > c->max_side)
    return fail(ESSL_E_CAPACITY, "image larger than context max_side");
  int max_radius = 0;
  bool any = false;
  int rc = check_aug(aug, n, &max_radius, &any);
  if (rc) return rc;
  if (max_radius) {
    rc = ensure_aug_scratch(c, (uint64_t)n * h * w * 3);
    if (rc) return rc;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const int r = pick_slot(c);
  if (r < 0) return r;
  std::memcpy(c->h_aug[r], aug, sizeof(essl_aug) * n);
  CK(cudaMemcpyAsync(c->d_aug[r], c->h_aug[r], sizeof(essl_aug) * n, cudaMemcpyHostToDevice, st));
  essl::AugOutParams ap{src, c->aug_b, c->d_aug[r], n, h, w, ESSL_OUT_NONE, nullptr, 0, dst};
  {
    Prof pr(c, ESSL_K_AUG, st);
    essl::launch_aug(ap, max_radius, st);
  }
  CK(cudaGetLastError());
  CK(cudaEventRecord(c->ev_desc[r], st));
  return ESSL_OK;
}

int essl_decode_crop_u8(essl_ctx *c, const uint8_t *blob, const essl_sample *samples, int n,
                        uint8_t *out, const uint64_t *out_offsets, essl_result *results,
                        void *stream) {
  if (!c || n < 0 || (n > 0 && (!blob || !samples || !out || !out_offsets)))
    return fail(ESSL_E_ARG, "essl_decode_crop_u8: bad arguments");
  DevGuard dg_(c);
  if (n == 0) return ESSL_OK;
  cudaStream_t st = (cudaStream_t)stream;
  int ring = -1;
  int rc = run_decode(c, blob, samples, n, results, st, &ring);
  if (rc) return rc;
  CK(cudaMemcpyAsync(c->d_offsets, out_offsets, sizeof(uint64_t) * n, cudaMemcpyHostToDevice, st));
  {
    Prof pr(c, ESSL_K_CROP, st);
    essl::launch_crop_u8(c->s.info, c->s.plane, n, out, c->d_offsets, st);
  }
  CK(cudaGetLastError());
  CK(cudaEventRecord(c->ev_desc[ring], st));
  CK(cudaStreamSynchronize(st));  // out_offsets is a host array
  return ESSL_OK;
}

int essl_dump_coefs(essl_ctx *c, const uint8_t *blob, const essl_sample *samples, int n,
                    int16_t *out, const uint64_t *out_offsets, int64_t out_cap, int32_t *geometry,
                    essl_result *results, void *stream) {
  if (!c || n < 0 || (n > 0 && (!blob || !samples || !out || !out_offsets || !geometry)))
    return fail(ESSL_E_ARG, "essl_dump_coefs: bad arguments");
  DevGuard dg_(c);
  if (n == 0) return ESSL_OK;
  cudaStream_t st = (cudaStream_t)stream;
  int ring = -1;
  int rc = run_decode(c, blob, samples, n, results, st, &ring);
  if (rc) return rc;
  std::vector<essl::ImgInfo> info(n);
  CK(cudaMemcpyAsync(info.data(), c->s.info, sizeof(essl::ImgInfo) * n, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  for (int i = 0; i < n; i++) {
    int64_t need = 0;
    for (int q = 0; q < 3; q++) {
      const bool ok = info[i].status == 0 && q < info[i].ncomp;
      geometry[i * 12 + 4 * q + 0] = ok ? info[i].wby0[q] : 0;
      geometry[i * 12 + 4 * q + 1] = ok ? info[i].wbx0[q] : 0;
      geometry[i * 12 + 4 * q + 2] = ok ? info[i].wbh[q] : 0;
      geometry[i * 12 + 4 * q + 3] = ok ? info[i].wbw[q] : 0;
      if (ok) need += (int64_t)info[i].wbh[q] * info[i].wbw[q] * 64;
    }
    if ((int64_t)out_offsets[i] + need > out_cap) return fail(ESSL_E_CAPACITY, "dump buffer too small");
  }
  CK(cudaMemcpyAsync(c->d_offsets, out_offsets, sizeof(uint64_t) * n, cudaMemcpyHostToDevice, st));
  {
    Prof pr(c, ESSL_K_DUMP, st);
    essl::launch_dump_coefs(c->s, n, out, c->d_offsets, st);
  }
  CK(cudaGetLastError());
  CK(cudaEventRecord(c->ev_desc[ring], st));
  CK(cudaStreamSynchronize(st));
  return ESSL_OK;
}

int essl_mask(essl_ctx *c, uint64_t seed, uint64_t epoch, const int64_t *index, int n, int tokens,
              int k, int32_t *mask_sorted, int64_t *ids_keep, int64_t *ids_restore, void *stream) {
  if (n < 0 || tokens < 1 || tokens > 4096 || k < 0 || k > tokens || (n > 0 && !index))
    return fail(ESSL_E_ARG, "essl_mask: bad arguments");
  DevGuard dg_(c);
  {
    Prof pr(c, ESSL_K_MASK, (cudaStream_t)stream);
    essl::launch_mask(seed, epoch, index, n, tokens, k, mask_sorted, ids_keep, ids_restore,
                      (cudaStream_t)stream);
  }
  CK(cudaGetLastError());
  return ESSL_OK;
}

int essl_mask_from_states(essl_ctx *c, const uint64_t *states, int n, int tokens, int k,
                          int32_t *mask_sorted, int64_t *ids_keep, int64_t *ids_restore,
                          void *stream) {
  if (n < 0 || tokens < 1 || tokens > 4096 || k < 0 || k > tokens || (n > 0 && !states))
    return fail(ESSL_E_ARG, "essl_mask_from_states: bad arguments");
  DevGuard dg_(c);
  {
    Prof pr(c, ESSL_K_MASK, (cudaStream_t)stream);
    essl::launch_mask_states(states, n, tokens, k, mask_sorted, ids_keep, ids_restore,
                             (cudaStream_t)stream);
  }
  CK(cudaGetLastError());
  return ESSL_OK;
}

int essl_gather_visible(essl_ctx *c, const void *pixels_bf16, int n, int res, int patch,
                        const int64_t *ids_keep, int n_keep, void *tokens_bf16, void *stream) {
  if (n < 0 || patch < 1 || res % patch || n_keep < 0 || (n > 0 && (!pixels_bf16 || !tokens_bf16)))
    return fail(ESSL_E_ARG, "essl_gather_visible: bad arguments");
  DevGuard dg_(c);
  {
    Prof pr(c, ESSL_K_GATHER, (cudaStream_t)stream);
    essl::launch_gather(pixels_bf16, n, res, patch, ids_keep, n_keep, tokens_bf16,
                        (cudaStream_t)stream);
  }
  CK(cudaGetLastError());
  return ESSL_OK;
}

int essl_resize_u8(const uint8_t *src, int ih, int iw, uint8_t *dst, int oh, int ow, int flip,
                   void *stream) {
  if (!src || !dst || ih < 1 || iw < 1 || oh < 1 || ow < 1)
    return fail(ESSL_E_ARG, "essl_resize_u8: bad arguments");
  essl::launch_resize_u8(src, ih, iw, dst, oh, ow, flip, (cudaStream_t)stream);
  CK(cudaGetLastError());
  return ESSL_OK;
}

int essl_normalize_u8(const uint8_t *src, int h, int w, float *dst, void *stream) {
  if (!src || !dst || h < 1 || w < 1) return fail(ESSL_E_ARG, "essl_normalize_u8: bad arguments");
  essl::launch_normalize_u8(src, h, w, dst, (cudaStream_t)stream);
  CK(cudaGetLastError());
  return ESSL_OK;
}


// ---- native batch enqueue ----------------------------------------------------

int essl_dataset_create(int64_t n, const uint64_t *offsets, const uint32_t *lengths,
                        const uint32_t *crc32, const uint16_t *widths, const uint16_t *heights,
                        const int64_t *labels, essl_dataset **out) {
  if (!out || n < 0 || (n > 0 && (!offsets || !lengths || !crc32 || !widths || !heights || !labels)))
    return fail(ESSL_E_ARG, "essl_dataset_create: bad arguments");
  essl_dataset *d = new essl_dataset();
  d->offset.assign(offsets, offsets + n);
  d->length.assign(lengths, lengths + n);
  d->crc.assign(crc32, crc32 + n);
  d->width.assign(widths, widths + n);
  d->height.assign(heights, heights + n);
  d->label.assign(labels, labels + n);
  *out = d;
  return ESSL_OK;
}

int essl_dataset_destroy(essl_dataset *d) {
  delete d;
  return ESSL_OK;
}

int essl_batch_enqueue(essl_ctx *c, const essl_dataset *ds, const essl_batch_cfg *cfg,
                       const int64_t *indices, int n, const essl_batch_io *io, void *stream) {
  if (!c || !ds || !cfg || !io || n < 0 || (n > 0 && !indices))
    return fail(ESSL_E_ARG, "essl_batch_enqueue: bad arguments");
  if (n > c->max_batch) return fail(ESSL_E_CAPACITY, "batch larger than context max_batch");
  if (!io->blob && !io->pinned_base) return fail(ESSL_E_ARG, "essl_batch_enqueue: no payload source");
  if (io->pinned_base && !io->blob && (io->stage_slot < 0 || io->stage_slot > 1))
    return fail(ESSL_E_ARG, "essl_batch_enqueue: bad staging slot");
  if (io->stage_chain < 0 || io->stage_chain > 1024)
    return fail(ESSL_E_ARG, "essl_batch_enqueue: bad stage_chain");
  if (cfg->tokens > 0 && (cfg->masked < 0 || cfg->masked > cfg->tokens || cfg->tokens > 4096))
    return fail(ESSL_E_ARG, "essl_batch_enqueue: bad mask geometry");
  if (io->tokens && cfg->tokens <= 0) return fail(ESSL_E_ARG, "visible tokens need the mask");
  const int64_t N = (int64_t)ds->offset.size();
  for (int i = 0; i < n; i++)
    if (indices[i] < 0 || indices[i] >= N) return fail(ESSL_E_ARG, "essl_batch_enqueue: index out of range");
  DevGuard dg_(c);
  if (n == 0) return ESSL_OK;
  NvtxRange nv_("essl_batch_enqueue");
  cudaStream_t st = (cudaStream_t)stream;
  if (io->wait_stream && io->wait_stream != stream) {
    CK(cudaEventRecord(c->ev_wait, (cudaStream_t)io->wait_stream));
    CK(cudaStreamWaitEvent(st, c->ev_wait, 0));
  }
  const int r = pick_slot(c);  // the batch that last used slot r has completed
  if (r < 0) return r;
  // descriptors: record fields + RRC rect and flip (host C++, pipeline.py:219-227)
  essl_sample *smp = c->h_desc[r];
  int64_t *il = c->h_il[r];
  for (int i = 0; i < n; i++) {
    const int64_t k = indices[i];
    smp[i].offset = ds->offset[k];
    smp[i].length = ds->length[k];
    smp[i].crc32 = ds->crc[k];
    smp[i].check_crc = cfg->check_crc;
    il[i] = k;
    il[n + i] = ds->label[k];
  }
  int rc = essl_rrc_batch(cfg->seed, cfg->epoch, indices, n, ds->width.data(), ds->height.data(),
                          cfg->scale[0], cfg->scale[1], cfg->ratio[0], cfg->ratio[1], smp);
  if (rc) return fail(rc, "essl_rrc_batch failed");
  if (io->index_label) {
    CK(cudaMemcpyAsync(io->index_label, il, 2 * sizeof(int64_t) * n, cudaMemcpyHostToDevice, st));
  }
  const uint8_t *blob = io->blob;
  if (!blob) {
    rc = stage_pinned_impl(c, io->stage_slot, io->pinned_base, smp, n, st, &blob, io->stage_chain);
    if (rc) return rc;
  }
  // MAE mask first: the fused visible-token output reads ids_restore
  if (cfg->tokens > 0) {
    if (!io->index_label) return fail(ESSL_E_ARG, "the mask needs the device index copy");
    Prof pr(c, ESSL_K_MASK, st);
    essl::launch_mask(cfg->seed, cfg->epoch, io->index_label, n, cfg->tokens, cfg->masked, io->mask,
                      io->ids_keep, io->ids_restore, st);
  }
  if (io->tokens && !io->ids_restore) return fail(ESSL_E_ARG, "visible tokens need ids_restore");
  rc = rrc_impl(c, blob, smp, r, io->aug, n, cfg->res, cfg->out_kind, io->pixels, io->pixel_stride,
                io->u8, cfg->patch, io->ids_restore, cfg->tokens - cfg->masked, io->tokens,
                io->results, st);
  if (rc) return rc;
  if (io->results_host && io->results)
    CK(cudaMemcpyAsync(io->results_host, io->results, sizeof(essl_result) * n, cudaMemcpyDeviceToHost, st));
  CK(cudaEventRecord(c->ev_desc[r], st));  // (again: covers the results copy)
  return ESSL_OK;
}

}  // extern "C"
