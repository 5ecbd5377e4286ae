// Runtime and C ABI of the B200 xGETT (include/gett_b200.h).
//
// Call path (mirrors kernel.py:124-155 _gett):
//   validate (planner.cpp, reference codes/order) -> return errors, C untouched
//   -> empty iteration space: return, nothing written (kernel.py:93-94)
//   -> plan (cached: folded M/N/K groups + device offset tables)
//   -> kernel choice: serial (aliasing C), ref-order, or tiled (DMMA / FFMA)
//   -> host path only: H2D of the addressed spans before, D2H of C's span after.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <list>
#include <memory>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/gett_b200.h"
#include "device.cuh"
#include "kernels.hpp"
#include "planner.hpp"

namespace gett {
namespace {

enum class Mode { Auto, Ref, Tiled, Serial, Ffma, Dot };

// Locks: g_plan_mu guards the plan cache and the last-call memo (short
// sections); each device has its own DevState::mu, held while a call issues
// work on that device, so calls on different devices run concurrently.  A
// multi-device call takes its devices' locks in ascending order.
std::mutex g_plan_mu;
std::once_flag g_env_once;
Mode g_mode = Mode::Auto;
int g_split = 0;
bool g_dgett_ws = true;  // DGETT: warp-specialised kernel (GETT_DGETT_WS=0: synchronous kernel)
bool g_stream_k = true;  // DGETT: persistent stream-K schedule when tiles > 1 wave and not whole waves (GETT_STREAM_K=0: off)
bool g_tma = true;        // SGETT: TMA-fed operands for affine views (GETT_TMA=0: cp.async gathers)
bool g_sk_small = true;    // DGETT: stream-K instead of split-K at 56-73 tiles (GETT_SK_SMALL=0: off)
bool g_complex_4x = false; // cgett/zgett tiled: four real GETTs instead of one embedded GETT (GETT_COMPLEX_EMBED=0)
bool g_pair = false;      // SGETT: CTA-pair kernel for narrow-N split-K shapes (GETT_PAIR=1: on)
bool g_dgett_tma = true;  // DGETT: TMA-fed operands for affine views (GETT_DGETT_TMA=0: cp.async gathers)
bool g_dgett_bulk = true; // DGETT: C += acc as bulk shared->global adds of 32-wide row runs (GETT_DGETT_BULK=0: red.add per element)
int g_wide = 1;           // SGETT wide CTA-pair kernel: 0 off, 1 automatic, 2 whenever it applies (GETT_WIDE)
bool g_wide_tail = true;  // wide kernel: a partial last wave (<= half the pair slots) runs as two K halves per tile (GETT_WIDE_TAIL=0: off)
bool g_wide_k16 = true;   // wide kernel: K-major operands as one 16-k SWIZZLE_64B box per k-block (GETT_WIDE_K16=0: two SW32 boxes)
int g_l2hint = 16;         // DGETT schedule / L2 policies (SkParams::l2hint; GETT_WS_L2HINT): 16 = serpentine k (c2 DRAM reads -8 %)
bool g_wide_mix = false;  // wide kernel: mixed split, one tf32 + one bf16 MMA per 8 k (GETT_WIDE_MIX=1; 4096^3 229 vs 236 TF:
                          // the kernel is bound by the TMA line rate of its 32-byte K-major boxes, not by the MMAs)
int g_kr = 1;             // SGETT k-run kernel: 0 off, 1 automatic, 2 whenever it applies (GETT_KR)
bool g_kr_pair = true;    // k-run kernel as CTA pairs (cta_group::2) when the tiling allows, two k runs per
                          // k-block when they fit (c5 back to back 34.6 vs 40.2 us; GETT_KR_PAIR=0: one CTA per tile)
}  // namespace
int g_launch_pdl = 1;     // programmatic dependent launches of the k-run SGETT kernel and the split-K reduce (GETT_PDL)
namespace {
int g_kr_slots = 2;       // k-run kernel: operand / TMEM ring depth wanted (GETT_KR_SLOTS)
int g_kr_krn = 2;         // k-run kernel: most k runs per k-block for CTA pairs (GETT_KR_KRN)
bool g_kr_mix = true;     // k-run kernel: mixed split, one tf32 + one bf16 MMA per 8 k (GETT_KR_MIX=0: three tf32 MMAs)
bool g_kr_fused = false;  // k-run split-K: reduce inside the kernel (GETT_KR_FUSED=1); default the
                          // separate reduce kernel (c5 from a CUDA graph: 33.2 vs 37.8 us fused)
int g_pipeline_slabs = -1;  // -1: automatic; 0/1: off; n: n slabs (GETT_PIPELINE)
int g_multi_stage = 0;      // multi-device split-K: 1 = stage partials by cudaMemcpyPeer instead of peer loads (GETT_MULTI_STAGE)
std::vector<int> g_devices;  // default device list of the host entry points (gett_set_devices; empty = current device)
thread_local std::string t_last_error;
thread_local const char* t_last_kernel = "none";
thread_local bool t_capturing = false;  // the current device call is being captured
std::atomic<int64_t> g_launches{0};

void read_env_once() {
  const char* k = std::getenv("GETT_KERNEL");
  if (k) gett_set_kernel(k);
  const char* s = std::getenv("GETT_SPLIT_K");
  if (s) g_split = std::atoi(s);
  const char* wsv = std::getenv("GETT_DGETT_WS");
  if (wsv) g_dgett_ws = std::atoi(wsv) != 0;
  const char* skv = std::getenv("GETT_STREAM_K");
  if (skv) g_stream_k = std::atoi(skv) != 0;
  const char* sks = std::getenv("GETT_SK_SMALL");
  if (sks) g_sk_small = std::atoi(sks) != 0;
  const char* ce = std::getenv("GETT_COMPLEX_EMBED");
  if (ce) g_complex_4x = std::atoi(ce) == 0;
  const char* dtv = std::getenv("GETT_DGETT_TMA");
  if (dtv) g_dgett_tma = std::atoi(dtv) != 0;
  const char* dbv = std::getenv("GETT_DGETT_BULK");
  if (dbv) g_dgett_bulk = std::atoi(dbv) != 0;
  const char* wdv = std::getenv("GETT_WIDE");
  if (wdv) g_wide = std::atoi(wdv);
  const char* l2v = std::getenv("GETT_WS_L2HINT");
  if (l2v) g_l2hint = std::atoi(l2v);
  const char* wtv = std::getenv("GETT_WIDE_TAIL");
  if (wtv) g_wide_tail = std::atoi(wtv) != 0;
  const char* wkv = std::getenv("GETT_WIDE_K16");
  if (wkv) g_wide_k16 = std::atoi(wkv) != 0;
  const char* wmv = std::getenv("GETT_WIDE_MIX");
  if (wmv) g_wide_mix = std::atoi(wmv) != 0;
  const char* krv = std::getenv("GETT_KR");
  if (krv) g_kr = std::atoi(krv);
  const char* krp = std::getenv("GETT_KR_PAIR");
  if (krp) g_kr_pair = std::atoi(krp) != 0;
  const char* pdl = std::getenv("GETT_PDL");
  if (pdl) g_launch_pdl = std::atoi(pdl) != 0;
  const char* krs = std::getenv("GETT_KR_SLOTS");
  if (krs) g_kr_slots = std::max(2, std::min(8, std::atoi(krs)));
  const char* krk = std::getenv("GETT_KR_KRN");
  if (krk) g_kr_krn = std::atoi(krk);
  const char* krm = std::getenv("GETT_KR_MIX");
  if (krm) g_kr_mix = std::atoi(krm) != 0;
  const char* krf = std::getenv("GETT_KR_FUSED");
  if (krf) g_kr_fused = std::atoi(krf) != 0;
  const char* pv = std::getenv("GETT_PAIR");
  if (pv) g_pair = std::atoi(pv) != 0;
  const char* tv = std::getenv("GETT_TMA");
  if (tv) g_tma = std::atoi(tv) != 0;
  const char* pl = std::getenv("GETT_PIPELINE");
  if (pl) g_pipeline_slabs = std::atoi(pl);
  const char* ms = std::getenv("GETT_MULTI_STAGE");
  if (ms) g_multi_stage = std::atoi(ms) != 0;
}
void read_env() { std::call_once(g_env_once, read_env_once); }

int cuda_fail(cudaError_t e, const char* what) {
  cudaGetLastError();  // clear a non-sticky error so the next call starts clean
  t_last_error = std::string(what) + ": " + cudaGetErrorString(e);
  return GETT_E_CUDA;
}

#define CK(expr)                                       \
  do {                                                 \
    cudaError_t e_ = (expr);                           \
    if (e_ != cudaSuccess) return cuda_fail(e_, #expr); \
  } while (0)

// Device-resident plan: offset tables for the groups.
struct DevPlan {
  Plan plan;
  int device = -1;
  int64_t* d_tab = nullptr;
  GroupDev gm{}, gn{}, gk{};
  int64_t* kref_a = nullptr;
  int64_t* kref_b = nullptr;
  int64_t* serial_tab = nullptr;
  int serial_nf = 0, serial_nc = 0;
  // residues used by the vector-load checks: every table entry divisible by 2 / 4
  bool am_even2 = false, am_even4 = false, ak_even2 = false, ak_even4 = false;
  bool bn_even2 = false, bn_even4 = false, bk_even2 = false, bk_even4 = false;
  // C offsets: every row offset even, and the N group's 32-aligned runs contiguous with even starts
  bool c_bulk_rows = false, c_bulk_cols = false;
  // SGETT TMA operand layouts (sgett_tc.cu): decided once per plan, tensor
  // maps re-encoded when the operand base pointers change
  int tma_state = 0;  // 0: not decided, 1: both operands TMA-fed, -1: gathers
  struct TmaLayout {
    uint64_t dims[5], strides[5];  // elements
    uint32_t box[5];
    int64_t base_off;              // element offset of coordinate 0
    TmaOperand op;
  } tma_l[2];
  TmaParams tma_p{};
  const void* tma_base[2] = {nullptr, nullptr};
  // the wide kernel's maps: K-major operands as one [16 k][128 rows]
  // SWIZZLE_64B box per k-block (half the TMA lines of two SW32 boxes)
  int tma64_state = 0;  // 0 undecided, 1 usable, -1 not
  TmaParams tma64_p{};
  const void* tma64_base[2] = {nullptr, nullptr};
  // CTA-pair SGETT on swapped roles (A2 = B' K-major, B2 = A' rows-major)
  int pair_state = 0;  // 0 undecided, 1 usable, -1 not
  TmaLayout pair_l[2];
  TmaParams pair_p{};
  const void* pair_base[2] = {nullptr, nullptr};
  GroupDev pgk{};      // dp.gk with its two tensors exchanged
  // SGETT k-run kernel (sgett_kr.cu): decided once per plan; the tensor maps
  // are re-encoded when the operand base pointers change
  // DGETT TMA layouts (dgett_ws.cu TMA path)
  int dtma_state = 0;  // 0 undecided, 1 both operands TMA-fed, -1 gathers
  TmaLayout dtma_l[2];
  TmaParams dtma_p{};
  const void* dtma_base[2] = {nullptr, nullptr};
  int kr_state = 0;    // 0 undecided, 1 usable, -1 not
  int kr_x = 0;        // X (TMEM operand) is the plan's A' (0) or B' (1)
  int kr_run = 0;      // KR
  struct KrLayout {
    uint64_t dims[5], strides[5];  // elements
    uint32_t box[5];
    int64_t base_off;
  } kr_l[2];            // X, Y
  KrParams kr_p{};
  const void* kr_base[2] = {nullptr, nullptr};
  // launch configurations: [0] one CTA per tile, one k run per k-block;
  // [1] CTA pairs (cta_group::2), two runs per k-block when they fit
  struct KrCfg {
    bool valid = false, pair = false;
    int krn = 1;
    KrParams kp{};       // slot / TMEM layout, tile counts (maps filled at launch)
    KrLayout lx, ly;     // the two tensor-map layouts
    CUtensorMap mx, my;
    const void* base[2] = {nullptr, nullptr};
  } krc[2];
  // used by a call captured into a CUDA graph: the graph holds raw pointers
  // into d_tab, so the LRU never evicts it (gett_release_caches still does)
  std::atomic<bool> pinned{false};
  ~DevPlan() {
    if (d_tab) {
      int cur = -1;
      cudaGetDevice(&cur);
      cudaSetDevice(device);
      cudaFree(d_tab);
      cudaSetDevice(cur);
    }
  }
};

struct PlanCache {
  std::list<std::string> lru;
  std::unordered_map<std::string, std::pair<std::shared_ptr<DevPlan>, std::list<std::string>::iterator>> map;
  static constexpr size_t kCap = 512;
};
PlanCache g_plans;

// drop least-recently-used plans beyond the cap, skipping plans pinned by a
// captured CUDA graph
void evict_plans() {
  auto it = g_plans.lru.end();
  while (g_plans.map.size() > PlanCache::kCap && it != g_plans.lru.begin()) {
    --it;
    auto m = g_plans.map.find(*it);
    if (m->second.first->pinned) continue;
    g_plans.map.erase(m);
    it = g_plans.lru.erase(it);
  }
}

// the last validated descriptor and its plan (gett_impl; under g_plan_mu)
struct LastCall {
  std::vector<int64_t> key;
  std::shared_ptr<DevPlan> dp;
} g_last;
thread_local std::vector<int64_t> t_key;  // the calling thread's descriptor key

struct Scratch {
  void* p = nullptr;
  size_t bytes = 0;
};
// Workspaces written by kernels are per stream: launches on different streams
// of one device may overlap.
struct StreamWs {
  Scratch ws;         // split-K partials
  Scratch part;       // stream-K tail partials
  Scratch flags;      // stream-K publish flags (zeroed on allocation)
  Scratch cx;         // real embedding of a complex operand
  int32_t epoch = 0;  // stream-K launches so far on this stream
  Scratch krsync;     // k-run kernel: tile counters, generations, slice claims (zeroed on allocation)
};
// A lane: one compute stream + two copy streams + the host path's device
// staging of one device.  Lane 0 serves single-device calls; a multi-device
// call that lists a device k times uses its lanes 0..k-1 (one GPU can stand in
// for several: the multi-device path is exercised with devices = (0, 0)).
struct Lane {
  cudaStream_t stream = nullptr;
  cudaStream_t h2d = nullptr, d2h = nullptr;  // copy streams of the pipelined host path
  std::vector<cudaEvent_t> events;
  Scratch a, b, c;
  Scratch red;  // multi-device split-K: staged partials of the other lanes
  cudaEvent_t event(size_t i) {
    while (events.size() <= i) {
      cudaEvent_t e = nullptr;
      if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return nullptr;
      events.push_back(e);
    }
    return events[i];
  }
};
struct DevState {
  std::mutex mu;
  std::unordered_map<cudaStream_t, StreamWs> sws;
  std::vector<std::unique_ptr<Lane>> lanes;
  int sms = 0;
};
constexpr int kMaxDevices = 64;
DevState g_dev[kMaxDevices];

int ensure(Scratch& s, size_t bytes) {
  if (bytes <= s.bytes) return 0;
  if (s.p) cudaFree(s.p);
  s.p = nullptr;
  s.bytes = 0;
  size_t want = bytes + bytes / 8 + 256;
  cudaError_t e = cudaMalloc(&s.p, want);
  if (e != cudaSuccess) {
    cudaGetLastError();
    t_last_error = std::string("cudaMalloc scratch: ") + cudaGetErrorString(e);
    return GETT_E_NOMEM;
  }
  s.bytes = want;
  return 0;
}

bool all_div(const std::vector<int64_t>& v, int64_t d) {
  for (int64_t x : v)
    if (x % d) return false;
  return true;
}

GroupDev to_dev(const Group& g, const int64_t* t0, const int64_t* t1) {
  GroupDev d;
  d.G = (int32_t)g.G;
  d.e_in = FastDiv::make((int32_t)g.e_in);
  d.s_in[0] = g.s_in[0];
  d.s_in[1] = g.s_in[1];
  d.T[0] = t0;
  d.T[1] = t1;
  return d;
}

// restatement of _plan_tables (plan.py:258-289) for the serial kernel
std::vector<int64_t> serial_table(const View& a, const View& b, const Spec& s, int* nf, int* nc) {
  int rank_c = a.rank + b.rank - 2 * s.conts;
  std::vector<int64_t> out_inc(rank_c), src_inc(rank_c), from_a(rank_c), ext_free(rank_c);
  int i = 0;
  auto contracted = [](const int64_t* idx, int n, int d) {
    for (int k = 0; k < n; ++k)
      if (idx[k] == d) return true;
    return false;
  };
  for (int d = 0; d < a.rank; ++d) {
    if (contracted(s.cont_a, s.conts, d)) continue;
    int64_t q = s.perm[i++];
    ext_free[q] = a.ext[d]; src_inc[q] = a.inc[d]; out_inc[q] = s.inc_c[q]; from_a[q] = 1;
  }
  for (int d = 0; d < b.rank; ++d) {
    if (contracted(s.cont_b, s.conts, d)) continue;
    int64_t q = s.perm[i++];
    ext_free[q] = b.ext[d]; src_inc[q] = b.inc[d]; out_inc[q] = s.inc_c[q]; from_a[q] = 0;
  }
  std::vector<int64_t> t;
  t.insert(t.end(), out_inc.begin(), out_inc.end());
  t.insert(t.end(), src_inc.begin(), src_inc.end());
  t.insert(t.end(), from_a.begin(), from_a.end());
  t.insert(t.end(), ext_free.begin(), ext_free.end());
  for (int k = 0; k < s.conts; ++k) t.push_back(a.inc[s.cont_a[k]]);
  for (int k = 0; k < s.conts; ++k) t.push_back(b.inc[s.cont_b[k]]);
  for (int k = 0; k < s.conts; ++k) t.push_back(a.ext[s.cont_a[k]]);
  *nf = rank_c;
  *nc = s.conts;
  return t;
}

int get_plan(char dtype, const View& a, const View& b, const Spec& s, int64_t off_c,
             int64_t len_c, std::shared_ptr<DevPlan>* out) {
  int dev = 0;
  CK(cudaGetDevice(&dev));
  std::string key = plan_key(dtype, a, b, s, off_c);
  key.append(reinterpret_cast<const char*>(&dev), sizeof dev);
  std::lock_guard<std::mutex> lock(g_plan_mu);
  auto it = g_plans.map.find(key);
  if (it != g_plans.map.end()) {
    g_plans.lru.splice(g_plans.lru.begin(), g_plans.lru, it->second.second);
    *out = it->second.first;
    if (t_capturing) (*out)->pinned = true;
    return 0;
  }
  auto dp = std::make_shared<DevPlan>();
  dp->pinned = t_capturing;
  dp->plan = build_plan(a, b, s, off_c, len_c);
  dp->device = dev;
  const Plan& p = dp->plan;
  if (p.gm.G >= (1LL << 31) || p.gn.G >= (1LL << 31) || p.gk.G >= (1LL << 31) ||
      p.rank_c > 64 || s.conts > 64) {
    t_last_error = "group extent >= 2^31 or rank > 64 is not supported";
    return GETT_E_UNSUPPORTED;
  }
  std::vector<int64_t> host;
  std::vector<size_t> offs;
  auto push = [&](const std::vector<int64_t>& v) {
    offs.push_back(host.size());
    host.insert(host.end(), v.begin(), v.end());
  };
  push(p.gm.T[0]); push(p.gm.T[1]);
  push(p.gn.T[0]); push(p.gn.T[1]);
  push(p.gk.T[0]); push(p.gk.T[1]);
  push(p.gk_ref.T[0]); push(p.gk_ref.T[1]);
  push(serial_table(a, b, s, &dp->serial_nf, &dp->serial_nc));
  CK(cudaMalloc(&dp->d_tab, host.size() * sizeof(int64_t)));
  CK(cudaMemcpy(dp->d_tab, host.data(), host.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
  int64_t* t = dp->d_tab;
  dp->gm = to_dev(p.gm, t + offs[0], t + offs[1]);
  dp->gn = to_dev(p.gn, t + offs[2], t + offs[3]);
  dp->gk = to_dev(p.gk, t + offs[4], t + offs[5]);
  dp->kref_a = t + offs[6];
  dp->kref_b = t + offs[7];
  dp->serial_tab = t + offs[8];
  dp->am_even2 = all_div(p.gm.T[0], 2); dp->am_even4 = all_div(p.gm.T[0], 4);
  dp->ak_even2 = all_div(p.gk.T[0], 2); dp->ak_even4 = all_div(p.gk.T[0], 4);
  dp->bn_even2 = all_div(p.gn.T[0], 2); dp->bn_even4 = all_div(p.gn.T[0], 4);
  dp->bk_even2 = all_div(p.gk.T[1], 2); dp->bk_even4 = all_div(p.gk.T[1], 4);
  dp->c_bulk_rows = all_div(p.gm.T[1], 2) && (p.gm.e_in == 1 || p.gm.s_in[1] % 2 == 0);
  dp->c_bulk_cols = all_div(p.gn.T[1], 2) && p.gn.s_in[1] == 1 && p.gn.e_in % 32 == 0;
  g_plans.lru.push_front(key);
  g_plans.map[key] = {dp, g_plans.lru.begin()};
  evict_plans();
  *out = dp;
  return 0;
}

// zero_view: the view folded as a single group (second tensor unused)
int get_view_plan(int rank, const int64_t* ext, const int64_t* inc, std::shared_ptr<DevPlan>* out) {
  int dev = 0;
  CK(cudaGetDevice(&dev));
  std::string key = "\x01zero|";
  for (int d = 0; d < rank; ++d) key += std::to_string(ext[d]) + "," + std::to_string(inc[d]) + ";";
  key += "#" + std::to_string(dev);
  std::lock_guard<std::mutex> lock(g_plan_mu);
  auto it = g_plans.map.find(key);
  if (it != g_plans.map.end()) {
    g_plans.lru.splice(g_plans.lru.begin(), g_plans.lru, it->second.second);
    *out = it->second.first;
    return 0;
  }
  auto dp = std::make_shared<DevPlan>();
  dp->device = dev;
  dp->plan.gm = fold_view(rank, ext, inc);
  if (dp->plan.gm.G >= (1LL << 31)) {
    t_last_error = "zero_view larger than 2^31 elements";
    return GETT_E_UNSUPPORTED;
  }
  const std::vector<int64_t>& T = dp->plan.gm.T[0];
  CK(cudaMalloc(&dp->d_tab, T.size() * sizeof(int64_t)));
  CK(cudaMemcpy(dp->d_tab, T.data(), T.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
  dp->gm = to_dev(dp->plan.gm, dp->d_tab, dp->d_tab);
  g_plans.lru.push_front(key);
  g_plans.map[key] = {dp, g_plans.lru.begin()};
  evict_plans();
  *out = dp;
  return 0;
}

inline int64_t iabs(int64_t x) { return x < 0 ? -x : x; }

// 16-byte vector loads along the fast dimension are legal when the fast
// group's inner mode is unit-stride with extent divisible by V, every other
// offset contribution is divisible by V, and the base is 16-byte aligned.
bool vec_ok(const GroupDev& fast, bool fast_tab_div, const GroupDev& slow, bool slow_tab_div,
            int V, const void* base) {
  if (fast.s_in[0] != 1 || fast.e_in.d % V != 0 || !fast_tab_div) return false;
  if (!(slow.e_in.d == 1 || slow.s_in[0] % V == 0) || !slow_tab_div) return false;
  return ((uintptr_t)base % 16) == 0;
}

// ---- TMA operand layouts for the SGETT kernel (device.cuh TmaParams) ----

struct AffDim {
  int64_t ext, stride;  // elements
};

// A group's offsets in tensor t as mixed-radix affine dims, inner first
// (extent-1 dims dropped): the inner mode (e_in, s_in) and the outer table
// decomposed greedily; false unless every table entry matches and every
// stride is positive.
bool affine_dims(const Group& g, int t, std::vector<AffDim>& d) {
  d.clear();
  if (g.e_in > 1) d.push_back({g.e_in, g.s_in[t]});
  const std::vector<int64_t>& T = g.T[t];
  const int64_t L = (int64_t)T.size();
  std::vector<AffDim> outer;
  int64_t pos = 1;
  while (pos < L) {
    const int64_t st = T[pos] - T[0];
    int64_t e = 1;
    while (pos * e < L && T[pos * e] - T[0] == e * st) ++e;
    if (L % (pos * e) != 0) return false;
    outer.push_back({e, st});
    pos *= e;
  }
  for (int64_t q = 0; q < L; ++q) {
    int64_t r = q, o = 0;
    for (const AffDim& a : outer) {
      o += (r % a.ext) * a.stride;
      r /= a.ext;
    }
    if (T[q] - T[0] != o) return false;
  }
  for (const AffDim& a : outer) d.push_back(a);
  for (const AffDim& a : d)
    if (a.stride <= 0) return false;
  return true;
}

// TMA layout of one operand: rows from group gr (tensor tr), k from gk
// (tensor tk).  K-major when the inner k mode is unit-stride (8-float SW32
// boxes), else rows-major when the inner row mode is; a 128-row tile must be
// one box (inner row extent a multiple of 128, or 128/e_in rows of the next
// dim, or a single tile).
bool tma_layout(const Group& gr, int tr, const Group& gk, int tk, DevPlan::TmaLayout& L, int tile = 128) {
  std::vector<AffDim> R, K;
  if (!affine_dims(gr, tr, R) || !affine_dims(gk, tk, K)) return false;
  if (R.empty() || K.empty() || R.size() > 3 || K.size() > 3) return false;
  if (K[0].ext % 8 != 0) return false;
  const bool kf = K[0].stride == 1;
  if (!kf && !(R[0].stride == 1 && R[0].ext % 4 == 0)) return false;
  const int64_t r0 = R[0].ext;
  int nrb;  // row dims carried by the box
  uint32_t rb[2] = {1, 1};
  if (r0 % tile == 0) {
    nrb = 1;
    rb[0] = (uint32_t)tile;
  } else if (tile % r0 == 0 && R.size() >= 2 && (R[1].ext % (tile / r0) == 0 || R.size() == 2)) {
    // (the last tile of a two-dim row group may run past the outer extent:
    // zero-filled, as rows past the view)
    nrb = 2;
    rb[0] = (uint32_t)r0;
    rb[1] = (uint32_t)(tile / r0);
  } else if (R.size() == 1) {
    nrb = 1;
    rb[0] = (uint32_t)tile;  // the last tile's rows past the extent are zero-filled
  } else {
    return false;
  }
  // box-carrying dims first (their order is the smem layout), then the rest
  // by ascending stride
  struct D {
    int64_t ext, stride;
    uint32_t box;
    int kind, idx;  // 0 row, 1 k
  };
  std::vector<D> dims, rest;
  if (kf) dims.push_back({K[0].ext, K[0].stride, 8u, 1, 0});
  for (int i = 0; i < nrb; ++i) dims.push_back({R[i].ext, R[i].stride, rb[i], 0, i});
  if (!kf) dims.push_back({K[0].ext, K[0].stride, 8u, 1, 0});
  for (size_t i = nrb; i < R.size(); ++i) rest.push_back({R[i].ext, R[i].stride, 1u, 0, (int)i});
  for (size_t i = 1; i < K.size(); ++i) rest.push_back({K[i].ext, K[i].stride, 1u, 1, (int)i});
  std::sort(rest.begin(), rest.end(), [](const D& x, const D& y) { return x.stride < y.stride; });
  for (const D& x : rest) dims.push_back(x);
  if (dims.size() > 5 || dims[0].stride != 1) return false;
  for (size_t i = 1; i < dims.size(); ++i)
    if (dims[i].stride % 4 != 0 || dims[i].stride * 4 >= (1LL << 40)) return false;
  std::memset(&L.op, 0, sizeof L.op);
  L.op.kf = kf ? 1 : 0;
  L.op.nr = (int32_t)R.size();
  L.op.nk = (int32_t)K.size();
  for (int i = 0; i < 5; ++i) {
    if (i < (int)dims.size()) {
      L.dims[i] = (uint64_t)dims[i].ext;
      L.strides[i] = (uint64_t)dims[i].stride;
      L.box[i] = dims[i].box;
      if (dims[i].kind == 0) {
        L.op.r_ext[dims[i].idx] = (int32_t)dims[i].ext;
        L.op.r_pos[dims[i].idx] = i;
      } else {
        L.op.k_ext[dims[i].idx] = (int32_t)dims[i].ext;
        L.op.k_pos[dims[i].idx] = i;
      }
    } else {
      L.dims[i] = 1;
      L.strides[i] = 4;
      L.box[i] = 1;
    }
  }
  L.base_off = gr.T[tr][0] + gk.T[tk][0];
  return true;
}

#ifndef GETT_TMA_PROMO
#define GETT_TMA_PROMO CU_TENSOR_MAP_L2_PROMOTION_L2_256B
#endif

typedef CUresult (*TmaEncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                CUtensorMapFloatOOBfill);

TmaEncodeFn tma_encode_fn() {
  static TmaEncodeFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&fn, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
  }
  return fn;
}

// k16: a K-major operand's boxes are 16 k wide with SWIZZLE_64B (the wide
// kernel) instead of 8 k with SWIZZLE_32B
bool tma_encode(const DevPlan::TmaLayout& L, const float* base, CUtensorMap* map, bool k16 = false) {
  TmaEncodeFn enc = tma_encode_fn();
  if (!enc) return false;
  const float* g = base + L.base_off;
  if ((uintptr_t)g % 16 != 0) return false;
  cuuint64_t dims[5], strides[4];
  cuuint32_t box[5], es[5] = {1, 1, 1, 1, 1};
  for (int i = 0; i < 5; ++i) {
    dims[i] = L.dims[i];
    box[i] = L.box[i];
    if (i) strides[i - 1] = L.strides[i] * 4;
  }
  CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_NONE;
  if (L.op.kf) {
    sw = k16 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B;
    if (k16) box[0] = 16;
  }
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, const_cast<float*>(g), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, sw, GETT_TMA_PROMO, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Both SGETT operands TMA-fed? (K a multiple of the 16-wide k-block; both
// layouts affine and encodable at these base pointers)
const TmaParams* sgett_tma(DevPlan& dp, const float* A, const float* B) {
  const Plan& p = dp.plan;
  if (dp.tma_state == 0) {
    dp.tma_state = -1;
    if (p.gk.G % 16 == 0 && p.gm.G > 1 && p.gn.G > 1 && tma_layout(p.gm, 0, p.gk, 0, dp.tma_l[0]) &&
        tma_layout(p.gn, 0, p.gk, 1, dp.tma_l[1]))
      dp.tma_state = 1;
    if (std::getenv("GETT_TMA_DEBUG")) {
      std::fprintf(stderr, "gett tma: %s\n", dp.tma_state == 1 ? "on" : "off");
      for (int t = 0; dp.tma_state == 1 && t < 2; ++t) {
        const DevPlan::TmaLayout& L = dp.tma_l[t];
        std::fprintf(stderr, "  op %d kf %d base_off %lld dims", t, L.op.kf, (long long)L.base_off);
        for (int i = 0; i < 5; ++i)
          std::fprintf(stderr, " (%llu,%llu,%u)", (unsigned long long)L.dims[i],
                       (unsigned long long)L.strides[i], L.box[i]);
        std::fprintf(stderr, "\n");
      }
    }
  }
  if (dp.tma_state != 1) return nullptr;
  if (dp.tma_base[0] != A || dp.tma_base[1] != B) {
    if (!tma_encode(dp.tma_l[0], A, &dp.tma_p.map[0]) || !tma_encode(dp.tma_l[1], B, &dp.tma_p.map[1])) {
      dp.tma_base[0] = dp.tma_base[1] = nullptr;
      return nullptr;
    }
    dp.tma_p.op[0] = dp.tma_l[0].op;
    dp.tma_p.op[1] = dp.tma_l[1].op;
    dp.tma_base[0] = A;
    dp.tma_base[1] = B;
  }
  return &dp.tma_p;
}

// The wide kernel's tensor maps: as sgett_tma, with every K-major operand
// loaded as one 16-k SWIZZLE_64B box per k-block (its inner k extent must be a
// multiple of 16).  Null when some K-major operand cannot (the caller then
// uses the SW32 maps).
const TmaParams* sgett_tma64(DevPlan& dp, const float* A, const float* B) {
  if (dp.tma_state != 1) return nullptr;
  if (dp.tma64_state == 0) {
    dp.tma64_state = 1;
    bool any = false;
    for (int t = 0; t < 2; ++t)
      if (dp.tma_l[t].op.kf) {
        any = true;
        if (dp.tma_l[t].dims[0] % 16 != 0) dp.tma64_state = -1;
      }
    if (!any) dp.tma64_state = -1;
  }
  if (dp.tma64_state != 1) return nullptr;
  if (dp.tma64_base[0] != A || dp.tma64_base[1] != B) {
    if (!tma_encode(dp.tma_l[0], A, &dp.tma64_p.map[0], true) ||
        !tma_encode(dp.tma_l[1], B, &dp.tma64_p.map[1], true)) {
      dp.tma64_base[0] = dp.tma64_base[1] = nullptr;
      return nullptr;
    }
    dp.tma64_p.op[0] = dp.tma_l[0].op;
    dp.tma64_p.op[1] = dp.tma_l[1].op;
    dp.tma64_base[0] = A;
    dp.tma64_base[1] = B;
  }
  return &dp.tma64_p;
}

// ---- SGETT k-run kernel (sgett_kr.cu) ----

// The K group as affine dims shared by both tensors, inner first: the inner
// mode, then the outer table cut wherever either tensor's offsets stop being
// one arithmetic progression.  False unless every entry matches.
bool joint_k_dims(const Group& gk, std::vector<int64_t>& ext, std::vector<int64_t> st[2]) {
  ext.clear();
  st[0].clear();
  st[1].clear();
  ext.push_back(gk.e_in);
  st[0].push_back(gk.s_in[0]);
  st[1].push_back(gk.s_in[1]);
  const std::vector<int64_t>& T0 = gk.T[0];
  const std::vector<int64_t>& T1 = gk.T[1];
  const int64_t L = (int64_t)T0.size();
  std::vector<int64_t> oe, os0, os1;
  int64_t pos = 1;
  while (pos < L) {
    const int64_t a = T0[pos] - T0[0], b = T1[pos] - T1[0];
    int64_t e = 1;
    while (pos * e < L && T0[pos * e] - T0[0] == e * a && T1[pos * e] - T1[0] == e * b) ++e;
    if (L % (pos * e) != 0) return false;
    oe.push_back(e);
    os0.push_back(a);
    os1.push_back(b);
    pos *= e;
  }
  for (int64_t q = 0; q < L; ++q) {
    int64_t r = q, o0 = 0, o1 = 0;
    for (size_t i = 0; i < oe.size(); ++i) {
      o0 += (r % oe[i]) * os0[i];
      o1 += (r % oe[i]) * os1[i];
      r /= oe[i];
    }
    if (T0[q] - T0[0] != o0 || T1[q] - T1[0] != o1) return false;
  }
  for (size_t i = 0; i < oe.size(); ++i) {
    ext.push_back(oe[i]);
    st[0].push_back(os0[i]);
    st[1].push_back(os1[i]);
  }
  return true;
}

// Box of up to `tile` rows over row dims R (inner first): how many dims it
// spans, their box extents and the rows it covers (a whole number of inner
// row runs when the inner extent is below `tile`: 50-row runs -> 100-row
// boxes); 0 when the rows cannot be boxed.
int row_box(const std::vector<AffDim>& R, int64_t tile, uint32_t* rb, int64_t* rows) {
  if (R.empty()) return 0;
  const int64_t r0 = R[0].ext;
  if (r0 >= tile || R.size() == 1) {
    rb[0] = (uint32_t)tile;
    *rows = tile;
    return 1;
  }
  const int64_t q = std::min<int64_t>(tile / r0, R[1].ext);
  rb[0] = (uint32_t)r0;
  rb[1] = (uint32_t)q;
  *rows = r0 * q;
  return 2;
}

// Decide (once per plan) whether the k-run kernel can run this SGETT, in
// which orientation, and build its two tensor-map layouts.
bool kr_decide(DevPlan& dp) {
  const Plan& p = dp.plan;
  std::vector<int64_t> kext, kst[2];
  if (!joint_k_dims(p.gk, kext, kst)) return false;
  for (int x = 0; x < 2; ++x) {
    const int y = 1 - x;
    const Group& gx = x == 0 ? p.gm : p.gn;
    const Group& gy = x == 0 ? p.gn : p.gm;
    if (kst[x][0] != 1 || kext[0] % 8 != 0) continue;
    // k run: the whole inner run when <= 64, else the largest multiple of 8
    // dividing it (the rest of the run becomes the innermost outer k digit)
    int64_t KR = kext[0];
    std::vector<int64_t> oe(kext.begin() + 1, kext.end()), os[2];
    os[0].assign(kst[0].begin() + 1, kst[0].end());
    os[1].assign(kst[1].begin() + 1, kst[1].end());
    if (KR > 64) {
      int64_t kr = 64;
      while (kr >= 8 && KR % kr) kr -= 8;
      if (kr < 8) continue;
      oe.insert(oe.begin(), KR / kr);
      os[0].insert(os[0].begin(), kr * kst[0][0]);
      os[1].insert(os[1].begin(), kr * kst[1][0]);
      KR = kr;
    }
    if (oe.size() > 2) continue;
    std::vector<AffDim> RX, RY;
    if (!affine_dims(gx, 0, RX) || !affine_dims(gy, 0, RY) || RX.empty() || RY.empty()) continue;
    if (RY[0].stride != 1) continue;  // Y rows-major
    bool pos_ok = kst[y][0] > 0;
    for (int t = 0; t < 2; ++t)
      for (int64_t v : os[t]) pos_ok = pos_ok && v > 0;
    if (!pos_ok) continue;
    const int64_t MX = gx.G, NY = gy.G;
    uint32_t xb[2] = {1, 1}, yb[2] = {1, 1};
    int64_t xrows = 0, yrows = 0;
    const int nxb = row_box(RX, 128, xb, &xrows);
    const int nyb = row_box(RY, NY <= 128 ? NY : 128, yb, &yrows);
    if (!nxb || !nyb || yrows % 4 != 0) continue;
    // one-dim boxes past the extent are zero-filled; a box of a multi-dim
    // row group must hold whole inner runs (checked by row_box) or start on
    // run boundaries (r0 a multiple of the box rows)
    if (nyb == 1 && RY.size() > 1 && RY[0].ext % yrows != 0) continue;
    if (nxb == 1 && RX.size() > 1 && RX[0].ext % xrows != 0) continue;
    const int64_t NT = (yrows + 15) / 16 * 16;
    const int nko = (int)oe.size();
    if (1 + (int)RX.size() + nko > 5 || (int)RY.size() + 1 + nko > 5) continue;
    struct D {
      int64_t ext, stride;
      uint32_t box;
    };
    std::vector<D> dx, dy;
    KrParams& kp = dp.kr_p;
    std::memset(&kp, 0, sizeof kp);
    // X: [k run][rows...][outer k...]
    dx.push_back({KR, 1, (uint32_t)(KR + 4)});  // (+4 zero-filled columns: conflict-free row pitch)
    for (size_t i = 0; i < RX.size(); ++i) {
      kp.xr_ext[i] = (int32_t)RX[i].ext;
      kp.xr_pos[i] = (int32_t)dx.size();
      dx.push_back({RX[i].ext, RX[i].stride, i < (size_t)nxb ? xb[i] : 1u});
    }
    // Y: [boxed rows][k run][other rows][outer k...]
    for (int i = 0; i < nyb; ++i) {
      kp.yr_ext[i] = (int32_t)RY[i].ext;
      kp.yr_pos[i] = (int32_t)dy.size();
      dy.push_back({RY[i].ext, RY[i].stride, yb[i]});
    }
    dy.push_back({KR, kst[y][0], (uint32_t)KR});
    for (size_t i = nyb; i < RY.size(); ++i) {
      kp.yr_ext[i] = (int32_t)RY[i].ext;
      kp.yr_pos[i] = (int32_t)dy.size();
      dy.push_back({RY[i].ext, RY[i].stride, 1u});
    }
    for (int j = 0; j < nko; ++j) {
      kp.k_ext[j] = (int32_t)oe[j];
      kp.xk_pos[j] = (int32_t)dx.size();
      dx.push_back({oe[j], os[x][j], 1u});
      kp.yk_pos[j] = (int32_t)dy.size();
      dy.push_back({oe[j], os[y][j], 1u});
    }
    bool ok = true;
    for (const std::vector<D>* dv : {&dx, &dy})
      for (size_t i = 1; i < dv->size(); ++i)
        ok = ok && (*dv)[i].stride % 4 == 0 && (*dv)[i].stride * 4 < (1LL << 40);
    if (!ok || dy[0].stride != 1) continue;
    for (int t = 0; t < 2; ++t) {
      const std::vector<D>& dv = t == 0 ? dx : dy;
      DevPlan::KrLayout& L = dp.kr_l[t];
      for (int i = 0; i < 5; ++i) {
        if (i < (int)dv.size()) {
          L.dims[i] = (uint64_t)dv[i].ext;
          L.strides[i] = (uint64_t)dv[i].stride;
          L.box[i] = dv[i].box;
        } else {
          L.dims[i] = 1;
          L.strides[i] = 4;
          L.box[i] = 1;
        }
      }
    }
    kp.xnr = (int32_t)RX.size();
    kp.ynr = (int32_t)RY.size();
    kp.nko = nko;
    kp.gx = x == 0 ? dp.gm : dp.gn;
    kp.gy = x == 0 ? dp.gn : dp.gm;
    kp.MX = (int32_t)MX;
    kp.NY = (int32_t)NY;
    kp.NT = (int32_t)NT;
    kp.x_rows = (int32_t)xrows;
    kp.y_rows = (int32_t)yrows;
    kp.tiles_x = (int32_t)((MX + xrows - 1) / xrows);
    kp.tiles_y = (int32_t)((NY + yrows - 1) / yrows);
    kp.nkb = (int32_t)(p.gk.G / KR);
    kp.kpc = 0;
    dp.kr_x = x;
    dp.kr_run = (int)KR;
    dp.kr_l[0].base_off = gx.T[0][0] + p.gk.T[x][0];
    dp.kr_l[1].base_off = gy.T[0][0] + p.gk.T[y][0];
    // launch configurations.  Shared memory: load slots [X raw 128 x (KR+4) |
    // Y raw KR x rows] of one k run each (freed right after the split) + two
    // operand slots [Y hi | Y lo] of a k-block = KRN runs (freed by the MMA) +
    // barriers, within 227 KB; TMEM: NT accumulator columns (rounded to 32) +
    // two A slots of 2 KE columns.  At least 2 KRN load slots keep the
    // mbarrier parity waits unambiguous (sgett_kr.cu, ring comment); one commit
    // frees a k-block's operand and TMEM slots (a second commit per k-block
    // costs ~46 clk of MMA issue, tools/mma_rate.cu).
    auto up = [](int64_t v, int64_t a) { return (v + a - 1) / a * a; };
    auto make = [&](DevPlan::KrCfg& c, int krn, bool pair) -> bool {
      c.valid = false;
      if (krn == 2 && (KR > 40 || nko < 1 || oe[0] % 2 != 0)) return false;
      if (pair && !(kp.tiles_x % 2 == 0 && yrows == NT && NT % 16 == 0 && nyb == 1)) return false;
      const int64_t KE = krn * KR, yr = pair ? NT / 2 : NT;
      KrParams q = kp;
      const int64_t xbytes = up(128 * (KR + 4) * 4, 1024), ybytes = up(KR * yr * 4, 128);
      q.lslot_bytes = (int32_t)(xbytes + ybytes);
      q.oslot_bytes = (int32_t)(2 * up(KE * yr * 4, 1024));
      q.a_col0 = (int32_t)up(NT, 32);
      auto fits = [&](int l, int o) {
        return (int64_t)l * q.lslot_bytes + (int64_t)o * q.oslot_bytes + 512 <= 227 * 1024;
      };
      // operand / TMEM ring depth: as deep as TMEM, shared memory and the load
      // ring allow (at most g_kr_slots): the split of k-block kb starts when the
      // MMAs of k-block kb - depth have finished, so a deeper ring keeps the
      // tensor pipe fed across the split warps' turnaround; load slots >= depth
      // x KRN keep the full-barrier parity waits unambiguous (sgett_kr.cu)
      int so = g_kr_slots;
      while (so > 2 && (q.a_col0 + so * 2 * KE > 512 || !fits(so * krn, so))) --so;
      if (q.a_col0 + so * 2 * KE > 512) return false;
      int sl = 8;
      while (sl > so * krn && !fits(sl, so)) --sl;
      if (!fits(sl, so)) return false;
      q.lslots = sl;
      q.oslots = so;
      q.aslots = so;
      q.o_off = sl * q.lslot_bytes;
      q.bar_off = (int32_t)(q.o_off + (int64_t)so * q.oslot_bytes);
      q.nkb = (int32_t)(p.gk.G / KE);
      c.kp = q;
      c.lx = dp.kr_l[0];
      c.ly = dp.kr_l[1];
      if (pair) c.ly.box[0] = (uint32_t)(NT / 2);
      c.krn = krn;
      c.pair = pair;
      c.base[0] = c.base[1] = nullptr;
      c.valid = true;
      return true;
    };
    if (!make(dp.krc[0], 1, false)) continue;
    if (g_kr_krn < 2 || !make(dp.krc[1], 2, true)) make(dp.krc[1], 1, true);
    return true;
  }
  return false;
}

bool kr_encode(const DevPlan::KrLayout& L, const float* base, CUtensorMap* map) {
  TmaEncodeFn enc = tma_encode_fn();
  if (!enc) return false;
  const float* g = base + L.base_off;
  if ((uintptr_t)g % 16 != 0) return false;
  cuuint64_t dims[5], strides[4];
  cuuint32_t box[5], es[5] = {1, 1, 1, 1, 1};
  for (int i = 0; i < 5; ++i) {
    dims[i] = L.dims[i];
    box[i] = L.box[i];
    if (i) strides[i - 1] = L.strides[i] * 4;
  }
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, const_cast<float*>(g), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, GETT_TMA_PROMO,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Run the SGETT on the k-run kernel when it applies.  Returns 1 when
// launched, 0 when the call does not fit, < 0 on error.
int try_sgett_kr(DevPlan& dp, const float* A, const float* B, float* C, int neg, cudaStream_t stream,
                 DevState& ds, StreamWs& sw) {
  if (g_kr == 0 || !g_tma) return 0;
  if (dp.kr_state == 0) {
    dp.kr_state = kr_decide(dp) ? 1 : -1;
    if (std::getenv("GETT_TMA_DEBUG")) {
      std::fprintf(stderr, "gett kr: %s", dp.kr_state == 1 ? "on" : "off");
      if (dp.kr_state == 1) {
        std::fprintf(stderr, " X=%s KR %d MX %d NY %d NT %d\n", dp.kr_x ? "B'" : "A'", dp.kr_run,
                     dp.kr_p.MX, dp.kr_p.NY, dp.kr_p.NT);
        for (int ci = 0; ci < 2; ++ci) {
          const DevPlan::KrCfg& c = dp.krc[ci];
          if (!c.valid) continue;
          std::fprintf(stderr, "  cfg %d: pair %d runs/k-block %d nkb %d slots load %d operand %d smem %d\n", ci,
                       (int)c.pair, c.krn, c.kp.nkb, c.kp.lslots, c.kp.oslots, c.kp.bar_off + 512);
          for (int t = 0; t < 2; ++t) {
            const DevPlan::KrLayout& L = t ? c.ly : c.lx;
            std::fprintf(stderr, "    %c base_off %lld dims", t ? 'Y' : 'X', (long long)L.base_off);
            for (int i = 0; i < 5; ++i)
              std::fprintf(stderr, " (%llu,%llu,%u)", (unsigned long long)L.dims[i],
                           (unsigned long long)L.strides[i], L.box[i]);
            std::fprintf(stderr, "\n");
          }
        }
      } else {
        std::fprintf(stderr, "\n");
      }
    }
  }
  if (dp.kr_state != 1) return 0;
  DevPlan::KrCfg& cfg = (g_kr_pair && dp.krc[1].valid) ? dp.krc[1] : dp.krc[0];
  KrParams kp = cfg.kp;
  const int64_t tiles = (int64_t)kp.tiles_x * kp.tiles_y;
  if (!ds.sms) {
    int dev = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&ds.sms, cudaDevAttrMultiProcessorCount, dev));
  }
  // automatic: the k-run kernel is for short runs (the SW32 boxes of the
  // tiled kernel issue one 32 B line per row per 8 k) and split-K shapes
  if (g_kr == 1 && !(dp.kr_run < 64 && tiles < ds.sms)) return 0;
  const float* X = dp.kr_x == 0 ? A : B;
  const float* Y = dp.kr_x == 0 ? B : A;
  if (cfg.base[0] != X || cfg.base[1] != Y) {
    if (!kr_encode(cfg.lx, X, &cfg.mx) || !kr_encode(cfg.ly, Y, &cfg.my)) {
      cfg.base[0] = cfg.base[1] = nullptr;
      return 0;
    }
    cfg.base[0] = X;
    cfg.base[1] = Y;
  }
  kp.mx = cfg.mx;
  kp.my = cfg.my;
  int64_t splits = 1;
  if (g_split > 0) splits = g_split;
  else if (tiles < ds.sms && kp.nkb >= 4) splits = ds.sms / tiles;
  if (splits > kp.nkb / 2) splits = kp.nkb / 2;
  if (splits > KR_MAX_SPLITS) splits = KR_MAX_SPLITS;  // (the fused reduce's claim slots)
  if (splits < 1) splits = 1;
  const int64_t kpc = (kp.nkb + splits - 1) / splits;
  splits = (kp.nkb + kpc - 1) / kpc;
  kp.kpc = (int32_t)kpc;
  kp.splits = (int32_t)splits;
  kp.C = C;
  kp.neg = neg;
  kp.cnt = kp.gen = kp.claim = nullptr;
  int rc;
  if (splits > 1) {
    if ((rc = ensure(sw.ws, (size_t)splits * kp.MX * kp.NY * sizeof(float)))) return rc;
    kp.ws = (float*)sw.ws.p;
    if (g_kr_fused && tiles <= KR_MAX_TILES) {
      // counters, generations and claims: zeroed once on allocation; they
      // return to a reusable state after every launch (graph replays too)
      // (a fixed layout for every call: counters [0, 256), generations
      // [256, 512), claims from 512 — slot t always belongs to tile t)
      const size_t bytes = (size_t)(2 * KR_MAX_TILES + KR_MAX_TILES * KR_MAX_SPLITS) * sizeof(uint32_t);
      if (sw.krsync.bytes < bytes) {
        if ((rc = ensure(sw.krsync, bytes))) return rc;
        CK(cudaMemsetAsync(sw.krsync.p, 0, sw.krsync.bytes, stream));
      }
      kp.cnt = (uint32_t*)sw.krsync.p;
      kp.gen = kp.cnt + KR_MAX_TILES;
      kp.claim = kp.gen + KR_MAX_TILES;
      static const int64_t spin =
          std::getenv("GETT_KR_SPIN_NS") ? std::atoll(std::getenv("GETT_KR_SPIN_NS")) : 200000;
      kp.spin_ns = spin;
    }
  }
  const bool pair = cfg.pair;
  const bool mix = g_kr_mix;
  CK(launch_sgett_kr(kp, dp.kr_run, cfg.krn, pair, mix, stream));
  ++g_launches;
#ifdef GETT_KR_NO_REDUCE  // tuning builds only: time the main kernel alone (wrong results)
  if (false) {
#else
  if (splits > 1 && kp.cnt == nullptr) {
#endif
    TiledParams<float> tp{};
    tp.C = C;
    tp.gm = kp.gx;
    tp.gn = kp.gy;
    tp.M = kp.MX;
    tp.N = kp.NY;
    tp.splits = kp.splits;
    tp.ws = kp.ws;
    tp.neg = neg;
    tp.ws_t = 1;
    CK(launch_splitk_reduce<float>(tp, stream));
    ++g_launches;
  }
  // [mix][pair][one pass, split-K, split-K reduced in the kernel]
  static const char* const kr_names[2][2][3] = {
      {{"sgett_tc3xtf32_kr", "sgett_tc3xtf32_kr_splitk", "sgett_tc3xtf32_kr_splitk_fused"},
       {"sgett_tc3xtf32_kr_pair", "sgett_tc3xtf32_kr_pair_splitk", "sgett_tc3xtf32_kr_pair_splitk_fused"}},
      {{"sgett_tctf32bf16_kr", "sgett_tctf32bf16_kr_splitk", "sgett_tctf32bf16_kr_splitk_fused"},
       {"sgett_tctf32bf16_kr_pair", "sgett_tctf32bf16_kr_pair_splitk", "sgett_tctf32bf16_kr_pair_splitk_fused"}}};
  t_last_kernel = kr_names[mix ? 1 : 0][pair ? 1 : 0][splits == 1 ? 0 : (kp.cnt ? 2 : 1)];
  return 1;
}

// ---- DGETT TMA layouts (dgett_ws.cu, TMA=true) ----
//
// Both operands of a DGETT tile are loaded as one box each per 32-deep
// k-block when their row and k groups are affine, into the same padded
// layouts the gathers write: a k-fast operand as [36 k | 128 rows] (smem
// [row][36]: the k run is cut into 32-wide digits, so k 32..35 of the box are
// out of bounds and zero-filled), a rows-fast one as [132 rows | 32 k] (smem
// [k][132]; its inner rows cut into 128-row digits, or one dim of at most 128
// rows).  The inner k run must hold whole 32-blocks and K be a multiple of
// 32, so no k-block straddles a digit of the K group and there is no K tail
// (its -0.0 padding stays with the gather path).

// one operand: rows from group gr (its tensor 0), k from the joint K dims
bool dgett_tma_layout(const Group& gr, const std::vector<int64_t>& kext, const std::vector<int64_t>& kst,
                      DevPlan::TmaLayout& L) {
  std::vector<AffDim> R;
  if (!affine_dims(gr, 0, R) || R.empty() || R.size() > 2) return false;
  for (const AffDim& d : R)
    if (d.stride <= 0) return false;
  for (size_t i = 0; i < kst.size(); ++i)
    if (kst[i] <= 0) return false;
  if (kext[0] % 32 != 0) return false;
  struct D {
    int64_t ext, stride;
    uint32_t box;
    int kind, idx;  // 0 row digit, 1 k digit
  };
  std::vector<D> dims;
  const bool kf = kst[0] == 1;
  if (kf) {
    // k digits: (32, 1) box 36, (kext0 / 32, 32), outer...; rows: a 128-row box
    dims.push_back({32, 1, 36u, 1, 0});
    if (R[0].ext % 128 == 0 || R.size() == 1) {
      dims.push_back({R[0].ext, R[0].stride, 128u, 0, 0});
      if (R.size() == 2) dims.push_back({R[1].ext, R[1].stride, 1u, 0, 1});
    } else if (128 % R[0].ext == 0) {
      dims.push_back({R[0].ext, R[0].stride, (uint32_t)R[0].ext, 0, 0});
      dims.push_back({R[1].ext, R[1].stride, (uint32_t)(128 / R[0].ext), 0, 1});
    } else {
      return false;
    }
    dims.push_back({kext[0] / 32, 32, 1u, 1, 1});
    for (size_t i = 1; i < kext.size(); ++i) dims.push_back({kext[i], kst[i], 1u, 1, (int)i + 1});
  } else {
    if (R[0].stride != 1) return false;
    // rows: (128, 1) box 132 [(R0 / 128, 128)] [R1]; k: kext0 box 32, outer...
    if (R[0].ext <= 128 && R.size() == 1) {
      dims.push_back({R[0].ext, 1, 132u, 0, 0});
      dims.push_back({kext[0], kst[0], 32u, 1, 0});
    } else if (R[0].ext % 128 == 0) {
      dims.push_back({128, 1, 132u, 0, 0});
      dims.push_back({kext[0], kst[0], 32u, 1, 0});
      dims.push_back({R[0].ext / 128, 128, 1u, 0, 1});
      if (R.size() == 2) dims.push_back({R[1].ext, R[1].stride, 1u, 0, 2});
    } else {
      return false;
    }
    for (size_t i = 1; i < kext.size(); ++i) dims.push_back({kext[i], kst[i], 1u, 1, (int)i});
  }
  if (dims.size() > 5) return false;
  for (size_t i = 1; i < dims.size(); ++i)
    if (dims[i].stride % 2 != 0 || dims[i].stride * 8 >= (1LL << 40)) return false;
  std::memset(&L.op, 0, sizeof L.op);
  L.op.kf = kf ? 1 : 0;
  int nr = 0, nk = 0;
  for (int i = 0; i < 5; ++i) {
    if (i < (int)dims.size()) {
      L.dims[i] = (uint64_t)dims[i].ext;
      L.strides[i] = (uint64_t)dims[i].stride;
      L.box[i] = dims[i].box;
      if (dims[i].kind == 0) {
        L.op.r_ext[dims[i].idx] = (int32_t)dims[i].ext;
        L.op.r_pos[dims[i].idx] = i;
        nr = std::max(nr, dims[i].idx + 1);
      } else {
        L.op.k_ext[dims[i].idx] = (int32_t)dims[i].ext;
        L.op.k_pos[dims[i].idx] = i;
        nk = std::max(nk, dims[i].idx + 1);
      }
    } else {
      L.dims[i] = 1;
      L.strides[i] = 2;
      L.box[i] = 1;
    }
  }
  if (nr > 3 || nk > 3) return false;
  L.op.nr = nr;
  L.op.nk = nk;
  return true;
}

bool dgett_tma_encode(const DevPlan::TmaLayout& L, const double* base, CUtensorMap* map) {
  TmaEncodeFn enc = tma_encode_fn();
  if (!enc) return false;
  const double* g = base + L.base_off;
  if ((uintptr_t)g % 16 != 0) return false;
  cuuint64_t dims[5], strides[4];
  cuuint32_t box[5], es[5] = {1, 1, 1, 1, 1};
  for (int i = 0; i < 5; ++i) {
    dims[i] = L.dims[i];
    box[i] = L.box[i];
    if (i) strides[i - 1] = L.strides[i] * 8;
  }
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, const_cast<double*>(g), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, GETT_TMA_PROMO,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Both DGETT operands TMA-fed?  Decided once per plan, tensor maps re-encoded
// when the base pointers change.  Returns null for the gather path.
const TmaParams* dgett_tma(DevPlan& dp, const double* A, const double* B) {
  const Plan& p = dp.plan;
  if (dp.dtma_state == 0) {
    dp.dtma_state = -1;
    std::vector<int64_t> kext, kst[2];
    if (p.gk.G % 32 == 0 && p.gm.G > 1 && p.gn.G > 1 && joint_k_dims(p.gk, kext, kst) &&
        dgett_tma_layout(p.gm, kext, kst[0], dp.dtma_l[0]) && dgett_tma_layout(p.gn, kext, kst[1], dp.dtma_l[1])) {
      dp.dtma_l[0].base_off = p.gm.T[0][0] + p.gk.T[0][0];
      dp.dtma_l[1].base_off = p.gn.T[0][0] + p.gk.T[1][0];
      dp.dtma_state = 1;
    }
    if (std::getenv("GETT_TMA_DEBUG")) {
      std::fprintf(stderr, "gett dgett tma: %s\n", dp.dtma_state == 1 ? "on" : "off");
      for (int t = 0; dp.dtma_state == 1 && t < 2; ++t) {
        const DevPlan::TmaLayout& L = dp.dtma_l[t];
        std::fprintf(stderr, "  op %d kf %d base_off %lld dims", t, L.op.kf, (long long)L.base_off);
        for (int i = 0; i < 5; ++i)
          std::fprintf(stderr, " (%llu,%llu,%u)", (unsigned long long)L.dims[i],
                       (unsigned long long)L.strides[i], L.box[i]);
        std::fprintf(stderr, "\n");
      }
    }
  }
  if (dp.dtma_state != 1) return nullptr;
  if (dp.dtma_base[0] != A || dp.dtma_base[1] != B) {
    if (!dgett_tma_encode(dp.dtma_l[0], A, &dp.dtma_p.map[0]) ||
        !dgett_tma_encode(dp.dtma_l[1], B, &dp.dtma_p.map[1])) {
      dp.dtma_base[0] = dp.dtma_base[1] = nullptr;
      return nullptr;
    }
    dp.dtma_p.op[0] = dp.dtma_l[0].op;
    dp.dtma_p.op[1] = dp.dtma_l[1].op;
    dp.dtma_base[0] = A;
    dp.dtma_base[1] = B;
  }
  return &dp.dtma_p;
}

// CTA-pair SGETT (sgett_tc.cu pair kernel) on the swapped roles: M2 = the
// plan's N (a K-major B', its rows 256 per pair in TMEM), N2 = the plan's M
// (a rows-major A' of <= 128 rows, split across the pair).  Returns 1 when
// launched, 0 when the call does not fit, < 0 on error.
int try_sgett_pair(DevPlan& dp, const float* A, const float* B, float* C, int neg, cudaStream_t stream,
                   DevState& ds, StreamWs& sw) {
  const Plan& p = dp.plan;
  if (!g_pair || !g_tma) return 0;
  const int64_t K = p.gk.G;
  if (dp.pair_state == 0) {
    // orientation 1 (swap): the K-major operand is the plan's B' (c5);
    // orientation 2: it is the plan's A'
    dp.pair_state = -1;
    for (int o = 1; o <= 2 && dp.pair_state < 0; ++o) {
      const Group& big = o == 1 ? p.gn : p.gm;    // rows of the K-major operand
      const Group& narrow = o == 1 ? p.gm : p.gn;
      const int tb = o == 1 ? 1 : 0, tn = o == 1 ? 0 : 1;  // their k tensors in gk
      if (K % 16 == 0 && big.G >= 256 && narrow.G <= 128 && narrow.G % 16 == 0 &&
          tma_layout(big, 0, p.gk, tb, dp.pair_l[0]) && dp.pair_l[0].op.kf == 1 &&
          tma_layout(narrow, 0, p.gk, tn, dp.pair_l[1], (int)(narrow.G / 2)) && dp.pair_l[1].op.kf == 0) {
        dp.pair_state = o;
        dp.pgk = dp.gk;
        if (o == 1) {
          std::swap(dp.pgk.T[0], dp.pgk.T[1]);
          std::swap(dp.pgk.s_in[0], dp.pgk.s_in[1]);
        }
      }
    }
  }
  if (dp.pair_state < 1) return 0;
  const bool sw1 = dp.pair_state == 1;
  const float* A2 = sw1 ? B : A;  // K-major operand (rows in TMEM)
  const float* B2 = sw1 ? A : B;  // narrow rows-major operand
  if (dp.pair_base[0] != A2 || dp.pair_base[1] != B2) {
    if (!tma_encode(dp.pair_l[0], A2, &dp.pair_p.map[0]) || !tma_encode(dp.pair_l[1], B2, &dp.pair_p.map[1])) {
      dp.pair_base[0] = dp.pair_base[1] = nullptr;
      return 0;
    }
    dp.pair_p.op[0] = dp.pair_l[0].op;
    dp.pair_p.op[1] = dp.pair_l[1].op;
    dp.pair_base[0] = A2;
    dp.pair_base[1] = B2;
  }
  if (!ds.sms) {
    int dev = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&ds.sms, cudaDevAttrMultiProcessorCount, dev));
  }
  const int64_t M2 = sw1 ? p.gn.G : p.gm.G, N2 = sw1 ? p.gm.G : p.gn.G;
  const int64_t pairs = (M2 + 255) / 256, kblocks = K / 16;
  int64_t splits = g_split > 0 ? g_split : ds.sms / (2 * pairs);
  if (splits > kblocks / 2) splits = kblocks / 2;
  if (splits < 1) splits = 1;
  const int64_t kchunk = ((kblocks + splits - 1) / splits) * 16;
  splits = (K + kchunk - 1) / kchunk;
  TiledParams<float> tp;
  tp.A = A2; tp.B = B2; tp.C = C;
  tp.gm = sw1 ? dp.gn : dp.gm;
  tp.gn = sw1 ? dp.gm : dp.gn;
  tp.gk = dp.pgk;
  tp.M = (int32_t)M2; tp.N = (int32_t)N2; tp.K = (int32_t)K;
  tp.tiles_m = (int32_t)pairs;  // (for the reduce: one column of tiles)
  tp.tiles_n = 1;
  tp.splits = (int32_t)splits;
  tp.k_chunk = (int32_t)kchunk;
  tp.neg = neg;
  tp.ws_t = 1;
  int rc = ensure(sw.ws, (size_t)splits * M2 * N2 * sizeof(float));
  if (rc) return rc;
  tp.ws = (float*)sw.ws.p;
  CK(launch_sgett_tc_pair(tp, dp.pair_p, stream));
  g_launches += 2;
  t_last_kernel = "sgett_tc3xtf32_pair_splitk";
  return 1;
}

// Self-overlapping C views run the literal reference loop on ONE GPU thread
// (their result depends on the reference's store order).  Legal but slow:
// warn once when a call is large enough to take seconds (> 2^26 MACs).
void warn_serial(int64_t size_free, int64_t size_cont) {
  static bool warned = false;
  if (warned || (double)size_free * (double)size_cont <= (double)(1LL << 26)) return;
  warned = true;
  std::fprintf(stderr,
               "gett: the C view overlaps itself (distinct coordinates share elements); its %lld x %lld "
               "MACs run in the reference's order on one GPU thread\n",
               (long long)size_free, (long long)size_cont);
}

template <typename T>
int run_device(DevPlan& dp, const T* a, const T* b, T* c, cudaStream_t stream, DevState& ds,
               int neg = 0, bool force_tiled = false) {
  const Plan& p = dp.plan;
  const T* A = p.swapped ? b : a;  // kernel roles A' / B'
  const T* B = p.swapped ? a : b;
  Mode mode = g_mode;
  if (force_tiled && mode != Mode::Ffma) mode = Mode::Tiled;  // complex real parts
  else if (p.c_may_alias) mode = Mode::Serial;
  const int64_t M = p.gm.G, N = p.gn.G, K = p.gk.G;
  if (mode == Mode::Auto) {
    if (K <= 8 || M * N * K <= (1LL << 18)) mode = Mode::Ref;
    else if (M * N <= (1LL << 14) && K >= 64 && M * N * K <= (1LL << 23)) mode = Mode::Dot;
    else mode = Mode::Tiled;
  }
  if (mode == Mode::Serial) {
    SerialParams<T> sp;
    sp.A = a; sp.B = b; sp.C = c;
    if (!dp.serial_tab) {
      t_last_error = "serial kernel requires an aliasing plan";
      return GETT_E_UNSUPPORTED;
    }
    sp.num_free = dp.serial_nf;
    sp.num_cont = dp.serial_nc;
    sp.size_free = p.size_free;
    sp.size_cont = p.size_cont;
    sp.tab = dp.serial_tab;
    warn_serial(p.size_free, p.size_cont);
    CK(launch_serial<T>(sp, stream));
    t_last_kernel = sizeof(T) == 8 ? "dgett_serial" : "sgett_serial";
    ++g_launches;
    return 0;
  }
  if (mode == Mode::Dot && K <= kDotStagedMaxK) {
    // staged-row dot kernel: stream the operand whose inner k mode is
    // unit-stride (or the smaller stride), stage the other
    DotParams<T> q;
    q.A = A; q.B = B; q.C = c;
    q.gm = dp.gm; q.gn = dp.gn; q.gk = dp.gk;
    q.M = (int32_t)M; q.N = (int32_t)N; q.K = (int32_t)K;
    q.stream_a = iabs(dp.gk.s_in[0]) <= iabs(dp.gk.s_in[1]) ? 1 : 0;
    CK(launch_dot_staged<T>(q, stream));
    t_last_kernel = sizeof(T) == 8 ? "dgett_dot" : "sgett_dot";
    ++g_launches;
    return 0;
  }
  if (mode == Mode::Ref || mode == Mode::Dot) {
    RefParams<T> rp;
    rp.A = A; rp.B = B; rp.C = c;
    rp.gm = dp.gm; rp.gn = dp.gn;
    rp.M = (int32_t)M; rp.N = (int32_t)N;
    rp.k_inner = (int32_t)p.gk_ref.e_in;
    rp.k_sa = p.gk_ref.s_in[0];
    rp.k_sb = p.gk_ref.s_in[1];
    rp.k_outer = (int32_t)p.gk_ref.T[0].size();
    rp.kta = dp.kref_a;
    rp.ktb = dp.kref_b;
    rp.kdiv = FastDiv::make(rp.k_inner);
    if (mode == Mode::Dot) {
      CK(launch_dot<T>(rp, stream));
      t_last_kernel = sizeof(T) == 8 ? "dgett_dot" : "sgett_dot";
    } else {
      CK(launch_ref<T>(rp, stream));
      t_last_kernel = sizeof(T) == 8 ? "dgett_ref_order" : "sgett_ref_order";
    }
    ++g_launches;
    return 0;
  }
  // tiled
  TiledParams<T> tp;
  tp.A = A; tp.B = B; tp.C = c;
  tp.gm = dp.gm; tp.gn = dp.gn; tp.gk = dp.gk;
  tp.M = (int32_t)M; tp.N = (int32_t)N; tp.K = (int32_t)K;
  // SGETT: 3xTF32 on tcgen05 unless forced to the FFMA core (or no k table)
  const bool use_tc = sizeof(T) == 4 && mode != Mode::Ffma;
  const int BM = use_tc ? tc_bm() : tiled_bm(), BN = use_tc ? tc_bn() : tiled_bn();
  const int BK = use_tc ? tc_bk() : tiled_bk((int)sizeof(T));
  tp.tiles_m = (int32_t)((M + BM - 1) / BM);
  tp.tiles_n = (int32_t)((N + BN - 1) / BN);
  int64_t tiles = (int64_t)tp.tiles_m * tp.tiles_n;
  int64_t kblocks = (K + BK - 1) / BK;
  int64_t splits = 1;
  // DGETT at 56-73 tiles: split-K would fill only 112-146 of the SMs with two
  // slices; stream-K shares (at most ~2.6 per tile) use all of them and skip
  // the reduce: 256 x 4096 x 4096 and 512 x 2048 x 4096 10 % faster.  Fewer
  // tiles cut each tile into more shares and lost (768 x 768 x 2048: -11 %).
  // (not under graph capture, where stream-K is off)
  // Under capture the shape takes one CTA per tile (no split-K either), so a
  // captured call needs no workspace its eager twin did not allocate.
  const bool sk_small_shape = sizeof(T) == 8 && g_dgett_ws && g_stream_k && g_sk_small &&
                              g_split <= 0 && tiles >= 56 && tiles < 74 && kblocks >= 16;
  bool sk_small = false;
  if (sk_small_shape) {
    cudaStreamCaptureStatus cap0 = cudaStreamCaptureStatusNone;
    CK(cudaStreamIsCapturing(stream, &cap0));
    sk_small = cap0 == cudaStreamCaptureStatusNone;
  }
  if (g_split > 0) splits = g_split;
  else if (tiles < 148 && kblocks >= 8 && !sk_small_shape) {
    splits = 148 / tiles;  // one wave of CTAs (1 CTA per SM for both tiled kernels)
    if (splits > kblocks / 2) splits = kblocks / 2;  // >= 2 k-blocks per slice
    if (splits < 1) splits = 1;
  }
  if (splits > kblocks) splits = kblocks;
  int64_t kchunk = ((kblocks + splits - 1) / splits) * BK;
  splits = (K + kchunk - 1) / kchunk;
  tp.k_chunk = (int32_t)kchunk;
  tp.splits = (int32_t)splits;
  tp.ws = nullptr;
  tp.neg = neg;
  tp.ws_t = use_tc ? 1 : 0;
  StreamWs& sw = ds.sws[stream];
  if (splits > 1) {
    int rc = ensure(sw.ws, (size_t)splits * M * N * sizeof(T));
    if (rc) return rc;
    tp.ws = (T*)sw.ws.p;
  }
  // gather directions and vector widths
  bool a_kf = dp.gk.e_in.d > 1 && (dp.gm.e_in.d == 1 || iabs(dp.gk.s_in[0]) < iabs(dp.gm.s_in[0]));
  bool b_kf = dp.gk.e_in.d > 1 && (dp.gn.e_in.d == 1 || iabs(dp.gk.s_in[1]) < iabs(dp.gn.s_in[0]));
  const int V = (int)(16 / sizeof(T));
  bool a_vec, b_vec;
  {
    GroupDev gkA = dp.gk;  // view gk from A''s side for the check
    GroupDev gkB = dp.gk;
    gkB.s_in[0] = dp.gk.s_in[1];
    bool akd = V == 2 ? dp.ak_even2 : dp.ak_even4;
    bool amd = V == 2 ? dp.am_even2 : dp.am_even4;
    bool bkd = V == 2 ? dp.bk_even2 : dp.bk_even4;
    bool bnd = V == 2 ? dp.bn_even2 : dp.bn_even4;
    a_vec = a_kf ? vec_ok(gkA, akd, dp.gm, amd, V, A) : vec_ok(dp.gm, amd, gkA, akd, V, A);
    b_vec = b_kf ? vec_ok(gkB, bkd, dp.gn, bnd, V, B) : vec_ok(dp.gn, bnd, gkB, bkd, V, B);
  }
  if (use_tc && sizeof(T) == 4) {
    const int kr = try_sgett_kr(dp, reinterpret_cast<const float*>(A), reinterpret_cast<const float*>(B),
                                reinterpret_cast<float*>(c), neg, stream, ds, sw);
    if (kr < 0) return kr;
    if (kr > 0) return 0;
  }
  if (use_tc && sizeof(T) == 4) {
    const int pr = try_sgett_pair(dp, reinterpret_cast<const float*>(A), reinterpret_cast<const float*>(B),
                                  reinterpret_cast<float*>(c), neg, stream, ds, sw);
    if (pr < 0) return pr;
    if (pr > 0) return 0;
  }
  if (use_tc) {
    const TmaParams* tma =
        g_tma ? sgett_tma(dp, reinterpret_cast<const float*>(A), reinterpret_cast<const float*>(B))
              : nullptr;
    if (tma) {
      a_kf = tma->op[0].kf != 0;
      b_kf = tma->op[1].kf != 0;
    }
    if (tma && g_wide > 0 && M >= 256 && N >= 256) {
      // wide CTA-pair kernel (256 x 256 per pair): half the shared-memory
      // traffic per MAC; automatic when the pair tiles fill at least half the
      // SMs without split-K, or K is long enough to split them
      if (!ds.sms) {
        int dev = 0;
        CK(cudaGetDevice(&dev));
        CK(cudaDeviceGetAttribute(&ds.sms, cudaDevAttrMultiProcessorCount, dev));
      }
      TiledParams<T> tw = tp;
      tw.tiles_m = (int32_t)((M + 255) / 256);
      tw.tiles_n = (int32_t)((N + 255) / 256);
      const int64_t pairs = (int64_t)tw.tiles_m * tw.tiles_n;
      const int64_t kb16 = K / 16;
      int64_t ws_split = g_split > 0 ? g_split : 1;
      if (g_split <= 0 && 2 * pairs < ds.sms && kb16 >= 64) {
        ws_split = ds.sms / (2 * pairs);
        if (ws_split > kb16 / 32) ws_split = kb16 / 32;  // >= 32 k-blocks per slice
        if (ws_split < 1) ws_split = 1;
      }
      const bool take = g_wide == 2 || (2 * pairs * ws_split >= ds.sms / 2 && kb16 >= 32);
      if (take) {
        int64_t kchunk = ((kb16 + ws_split - 1) / ws_split) * 16;
        ws_split = (K + kchunk - 1) / kchunk;
        tw.ws = nullptr;
        tw.ws_t = 1;
        // tail split: a partial last wave of at most half the pair slots runs
        // as two K halves per tile (3.46 -> 3.5 waves' time instead of 4 for
        // 4096^3); their partials go to a compact workspace
        const int64_t slots = ds.sms / 2, rem = pairs % slots;
        if (g_wide_tail && g_split <= 0 && ws_split == 1 && pairs > slots && rem > 0 && 2 * rem <= slots &&
            kb16 >= 64) {
          tw.tail_tile0 = (int32_t)(pairs - rem);
          tw.tail_tiles = (int32_t)rem;
          kchunk = ((kb16 + 1) / 2) * 16;
          int rc = ensure(sw.ws, (size_t)2 * rem * 65536 * sizeof(T));
          if (rc) return rc;
          tw.ws = (T*)sw.ws.p;
        }
        tw.k_chunk = (int32_t)kchunk;
        tw.splits = (int32_t)ws_split;
        if (ws_split > 1) {
          int rc = ensure(sw.ws, (size_t)ws_split * M * N * sizeof(T));
          if (rc) return rc;
          tw.ws = (T*)sw.ws.p;
        }
        const TmaParams* t64 = g_wide_k16 ? sgett_tma64(dp, reinterpret_cast<const float*>(A),
                                                        reinterpret_cast<const float*>(B))
                                          : nullptr;
        CK(launch_sgett_tc_wide(*reinterpret_cast<TiledParams<float>*>(&tw), t64 ? *t64 : *tma, a_kf, b_kf,
                                g_wide_mix, t64 != nullptr, stream));
        g_launches += (ws_split > 1 || tw.tail_tiles > 0) ? 2 : 1;
        if (g_wide_mix)
          t_last_kernel = ws_split > 1 ? "sgett_tctf32bf16_wide_splitk"
                                       : (tw.tail_tiles > 0 ? "sgett_tctf32bf16_wide_tail" : "sgett_tctf32bf16_wide");
        else
          t_last_kernel = ws_split > 1 ? "sgett_tc3xtf32_wide_splitk"
                                       : (tw.tail_tiles > 0 ? "sgett_tc3xtf32_wide_tail" : "sgett_tc3xtf32_wide");
        return 0;
      }
    }
    CK(launch_sgett_tc(*reinterpret_cast<TiledParams<float>*>(&tp), tma, a_kf, b_kf, a_vec, b_vec,
                       stream));
    g_launches += splits > 1 ? 2 : 1;
    t_last_kernel = tma ? (splits > 1 ? "sgett_tc3xtf32_tma_splitk" : "sgett_tc3xtf32_tma")
                        : (splits > 1 ? "sgett_tc3xtf32_splitk" : "sgett_tc3xtf32");
    return 0;
  }
  if (sizeof(T) == 8 && g_dgett_ws) {
    SkParams sk;
    sk.l2hint = g_l2hint;
    if (!ds.sms) {
      int dev = 0;
      CK(cudaGetDevice(&dev));
      CK(cudaDeviceGetAttribute(&ds.sms, cudaDevAttrMultiProcessorCount, dev));
    }
    const int64_t G = ds.sms;
    // (not inside a CUDA-graph capture: replays would reuse the publish epoch)
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    CK(cudaStreamIsCapturing(stream, &cap));
    if (g_stream_k && cap == cudaStreamCaptureStatusNone && splits == 1 && tiles % G != 0 &&
        (2 * tiles > G || sk_small)) {
      // persistent: the last 1-2 waves of tiles (all of them below 2 waves)
      // are shared out by k-block units, the rest run data-parallel; below one
      // wave (G/2 < tiles < G, where split-K cannot help) the shares are
      // shorter than a tile and the heads add several parts
      const int64_t waves = (tiles + G - 1) / G;
      sk.enabled = 1;
      sk.grid = (int32_t)G;
      sk.nkb = dgett_ws_tiles_k((int)K);
      sk.sk_tile0 = (int32_t)((waves < 2 ? 0 : waves - 2) * G);
      sk.sk_units = (tiles - sk.sk_tile0) * sk.nkb;
      int rc = ensure(sw.part, (size_t)G * 128 * 128 * sizeof(double));
      if (rc) return rc;
      const size_t fbytes = (size_t)G * sizeof(int32_t);
      if (sw.flags.bytes < fbytes) {
        if ((rc = ensure(sw.flags, fbytes))) return rc;
        CK(cudaMemsetAsync(sw.flags.p, 0, sw.flags.bytes, stream));
      }
      if (++sw.epoch <= 0) sw.epoch = 1;
      sk.part = (double*)sw.part.p;
      sk.flags = (int32_t*)sw.flags.p;
      sk.epoch = sw.epoch;
    }
    // C += acc as bulk adds of whole 32-wide row runs staged in shared memory
    tp.c_bulk = 0;
    if (g_dgett_bulk && dp.c_bulk_rows && dp.c_bulk_cols && (reinterpret_cast<uintptr_t>(c) & 15) == 0) {
      tp.c_bulk = 1;
      if (dp.gm.e_in.d % 32 == 0) tp.c_bulk |= 2;
    }
    const TmaParams* dtp =
        g_tma && g_dgett_tma ? dgett_tma(dp, reinterpret_cast<const double*>(A), reinterpret_cast<const double*>(B))
                             : nullptr;
    if (dtp) {
      a_kf = dtp->op[0].kf != 0;
      b_kf = dtp->op[1].kf != 0;
    }
    CK(launch_dgett_ws(*reinterpret_cast<TiledParams<double>*>(&tp), sk, dtp, a_kf, b_kf, a_vec,
                       b_vec, stream));
    g_launches += splits > 1 ? 2 : 1;
    // [tma][schedule: one CTA per tile, stream-K, split-K][bulk-add epilogue]
    static const char* const names[2][3][2] = {
        {{"dgett_dmma_ws", "dgett_dmma_ws_bulk"}, {"dgett_dmma_ws_sk", "dgett_dmma_ws_sk_bulk"},
         {"dgett_dmma_ws_splitk", "dgett_dmma_ws_splitk"}},
        {{"dgett_dmma_ws_tma", "dgett_dmma_ws_tma_bulk"}, {"dgett_dmma_ws_tma_sk", "dgett_dmma_ws_tma_sk_bulk"},
         {"dgett_dmma_ws_tma_splitk", "dgett_dmma_ws_tma_splitk"}}};
    t_last_kernel = names[dtp ? 1 : 0][splits > 1 ? 2 : sk.enabled ? 1 : 0][tp.c_bulk ? 1 : 0];
    return 0;
  }
  CK(launch_tiled<T>(tp, a_kf, b_kf, a_vec, b_vec, stream));
  g_launches += splits > 1 ? 2 : 1;
  t_last_kernel = sizeof(T) == 8 ? (splits > 1 ? "dgett_dmma_splitk" : "dgett_dmma")
                                 : (splits > 1 ? "sgett_ffma_splitk" : "sgett_ffma");
  return 0;
}

constexpr int kNotPipelined = 1 << 30;

// RAII: restore the caller's current device.
struct DeviceGuard {
  int dev = -1;
  DeviceGuard() { cudaGetDevice(&dev); }
  ~DeviceGuard() {
    if (dev >= 0) cudaSetDevice(dev);
  }
};

// Lane `i` of the current device's state (created on first use).  The caller
// holds ds.mu.
int get_lane(int dev, size_t i, Lane** out) {
  DevState& ds = g_dev[dev];
  while (ds.lanes.size() <= i) ds.lanes.emplace_back(new Lane());
  Lane& L = *ds.lanes[i];
  if (!L.stream) CK(cudaStreamCreateWithFlags(&L.stream, cudaStreamNonBlocking));
  if (!L.h2d) CK(cudaStreamCreateWithFlags(&L.h2d, cudaStreamNonBlocking));
  if (!L.d2h) CK(cudaStreamCreateWithFlags(&L.d2h, cudaStreamNonBlocking));
  *out = &L;
  return 0;
}

int current_device(int* dev) {
  CK(cudaGetDevice(dev));
  if (*dev < 0 || *dev >= kMaxDevices) {
    t_last_error = "device ordinal >= 64";
    return GETT_E_UNSUPPORTED;
  }
  return 0;
}

int event_at(Lane& L, size_t i, cudaEvent_t* e) {
  *e = L.event(i);
  if (!*e) {
    t_last_error = "cudaEventCreate failed";
    return GETT_E_CUDA;
  }
  return 0;
}

// The free mode that cuts an xGETT into slabs with disjoint C spans: among
// free modes of extent > 1, the one with the largest |C increment| (outermost
// in C), provided that increment exceeds the span of all other C modes.  A
// slab (rows [lo, hi) of that mode) is itself an xGETT on sub-views — a
// free-mode slice, bitwise equal to the same elements of the whole call — and
// xGETT calls whose C footprints are disjoint may run concurrently
// (SPEC.md:249).  This is the device-sharding rule of SURVEY §8e and the host
// pipeline's cut.
struct SlabCut {
  int owner = -1, dim = -1, q = -1;  // operand (0 = A, 1 = B), its dim, C position
  int64_t E = 0;                     // extent of the mode
  // the owner operand's slab spans are disjoint too (its stride of the mode
  // exceeds the span of its other modes): a slab uploads only its share of
  // the owner.  Otherwise (c5: the cut mode is B's innermost) every slab's
  // owner span is nearly the whole operand.
  bool owner_disjoint = false;
};

bool slab_cut(const Plan& p, const View& a, const View& b, const Spec& s, SlabCut* out) {
  auto contracted = [](const int64_t* idx, int n, int d) {
    for (int k = 0; k < n; ++k)
      if (idx[k] == d) return true;
    return false;
  };
  SlabCut c;
  int i = 0;
  int64_t best = -1;
  for (int t = 0; t < 2; ++t) {
    const View& v = t == 0 ? a : b;
    const int64_t* cont = t == 0 ? s.cont_a : s.cont_b;
    for (int d = 0; d < v.rank; ++d) {
      if (contracted(cont, s.conts, d)) continue;
      int qq = (int)s.perm[i++];
      if (v.ext[d] > 1 && iabs(s.inc_c[qq]) > best) {
        best = iabs(s.inc_c[qq]);
        c.owner = t; c.dim = d; c.q = qq; c.E = v.ext[d];
      }
    }
  }
  if (c.owner < 0) return false;
  int64_t other = 0;
  for (int qq = 0; qq < p.rank_c; ++qq)
    if (qq != c.q && p.ext_c[qq] > 0) other += iabs(s.inc_c[qq]) * (p.ext_c[qq] - 1);
  if (iabs(s.inc_c[c.q]) <= other) return false;
  const View& ov = c.owner == 0 ? a : b;
  int64_t ospan = 0;
  for (int d = 0; d < ov.rank; ++d)
    if (d != c.dim && ov.ext[d] > 0) ospan += iabs(ov.inc[d]) * (ov.ext[d] - 1);
  c.owner_disjoint = iabs(ov.inc[c.dim]) > ospan;
  *out = c;
  return true;
}

// Sub-views of rows [lo, hi) of the cut mode (the ext vectors own the arrays
// the views point at).
struct SlabViews {
  std::vector<int64_t> ext_o, ext_c;
  View a, b;
  int64_t off_c = 0;
  SlabViews(const SlabCut& cut, const View& va, const View& vb, const Spec& s, const Plan& p,
            int64_t off_c0, int64_t lo, int64_t hi)
      : ext_o(cut.owner == 0 ? va.ext : vb.ext, (cut.owner == 0 ? va.ext : vb.ext) + (cut.owner == 0 ? va.rank : vb.rank)),
        ext_c(p.ext_c), a(va), b(vb) {
    ext_o[cut.dim] = hi - lo;
    ext_c[cut.q] = hi - lo;
    if (cut.owner == 0) { a.ext = ext_o.data(); a.off = va.off + lo * va.inc[cut.dim]; }
    else { b.ext = ext_o.data(); b.off = vb.off + lo * vb.inc[cut.dim]; }
    off_c = off_c0 + lo * s.inc_c[cut.q];
  }
};

// Slab boundaries of rows [r0, r1) in S slabs: the last two are short (1 and
// 2 granules of 128 rows, or rows when the range is small) so that little
// compute and D2H is left after the last H2D (small slabs run split-K across
// the SMs); the rest are uniform, on granule boundaries.
std::vector<int64_t> slab_bounds(int64_t r0, int64_t r1, int64_t S) {
  const int64_t E = r1 - r0;
  std::vector<int64_t> bnd(S + 1);
  const int64_t g = E >= 16 * 128 ? 128 : 1;
  const int64_t R = E - 3 * g;
  if (S >= 4 && R >= (S - 2) * g) {
    for (int64_t i = 0; i <= S - 2; ++i) bnd[i] = (R * i / (S - 2)) / g * g;
    bnd[S - 2] = R;
    bnd[S - 1] = R + 2 * g;
    bnd[S] = E;
  } else {
    for (int64_t i = 0; i <= S; ++i) bnd[i] = E * i / S;
  }
  for (auto& x : bnd) x += r0;
  return bnd;
}

// Issue (no synchronisation) rows [r0, r1) of the cut mode as S slabs on one
// lane: per slab, H2D of the owner operand's and C's slab spans on L.h2d, the
// kernel on L.stream, D2H of C's slab span on L.d2h — slab s computes while
// slab s+1 is copied in and slab s-1 is copied out.  base_x mirror host
// element indices over the whole call's spans; the non-owning operand must
// already be queued on L.h2d (or be in place).  Events from index ev0 on.
template <typename T>
int issue_slabs(Lane& L, DevState& ds, const SlabCut& cut, const View& a, const View& b,
                const Spec& s, const Plan& p, const T* ha, const T* hb, T* hc, int64_t off_c,
                int64_t len_c, int64_t r0, int64_t r1, int64_t S, T* base_a, T* base_b,
                T* base_c, size_t ev0) {
  const std::vector<int64_t> bnd = slab_bounds(r0, r1, S);
  for (int64_t sl = 0; sl < S; ++sl) {
    if (bnd[sl + 1] == bnd[sl]) continue;
    SlabViews v(cut, a, b, s, p, off_c, bnd[sl], bnd[sl + 1]);
    std::shared_ptr<DevPlan> dp;
    int rc = get_plan(sizeof(T) == 8 ? 'd' : 's', v.a, v.b, s, v.off_c, len_c, &dp);
    if (rc) return rc;
    int64_t flo, fhi;
    const View& so = cut.owner == 0 ? v.a : v.b;
    footprint(so.rank, so.ext, so.inc, &flo, &fhi);
    const int64_t olo = so.off + flo;
    const size_t on = (size_t)(fhi - flo + 1);
    T* obase = cut.owner == 0 ? base_a : base_b;
    const T* ohost = cut.owner == 0 ? ha : hb;
    CK(cudaMemcpyAsync(obase + olo, ohost + olo, on * sizeof(T), cudaMemcpyHostToDevice, L.h2d));
    footprint(p.rank_c, v.ext_c.data(), s.inc_c, &flo, &fhi);
    const int64_t clo = v.off_c + flo;
    const size_t cn = (size_t)(fhi - flo + 1);
    CK(cudaMemcpyAsync(base_c + clo, hc + clo, cn * sizeof(T), cudaMemcpyHostToDevice, L.h2d));
    cudaEvent_t ein, eout;
    if ((rc = event_at(L, ev0 + 2 * sl, &ein)) || (rc = event_at(L, ev0 + 2 * sl + 1, &eout))) return rc;
    CK(cudaEventRecord(ein, L.h2d));
    CK(cudaStreamWaitEvent(L.stream, ein, 0));
    rc = run_device<T>(*dp, base_a + v.a.off, base_b + v.b.off, base_c + v.off_c, L.stream, ds);
    if (rc) return rc;
    CK(cudaEventRecord(eout, L.stream));
    CK(cudaStreamWaitEvent(L.d2h, eout, 0));
    CK(cudaMemcpyAsync(hc + clo, base_c + clo, cn * sizeof(T), cudaMemcpyDeviceToHost, L.d2h));
  }
  return 0;
}

// Host-buffer path with transfers overlapped (one device): C's outermost
// free mode is cut into slabs (issue_slabs); the operand that does not own the
// slab mode is copied once, up front.
template <typename T>
int host_pipelined(DevPlan& full, const View& a, const View& b, const Spec& s, const T* ha,
                   const T* hb, T* hc, int64_t off_c, int64_t len_c, DevState& ds, Lane& L) {
  const Plan& p = full.plan;
  if (g_pipeline_slabs == 0 || g_pipeline_slabs == 1 || p.c_may_alias) return kNotPipelined;
  const size_t na = (size_t)(p.fp_hi[0] - p.fp_lo[0] + 1);
  const size_t nb = (size_t)(p.fp_hi[1] - p.fp_lo[1] + 1);
  const size_t nc = (size_t)(p.fp_hi[2] - p.fp_lo[2] + 1);
  if (g_pipeline_slabs < 0 && (na + nb + 2 * nc) * sizeof(T) < (64u << 20)) return kNotPipelined;
  SlabCut cut;
  if (!slab_cut(p, a, b, s, &cut) || (!cut.owner_disjoint && g_pipeline_slabs < 0)) return kNotPipelined;
  int64_t S = g_pipeline_slabs > 1 ? g_pipeline_slabs : 10;  // c2: 8 -> 8.66, 10 -> 8.43 ms
  if (S > cut.E) S = cut.E;
  if (S < 2) return kNotPipelined;
  int rc;
  if ((rc = ensure(L.a, na * sizeof(T))) || (rc = ensure(L.b, nb * sizeof(T))) ||
      (rc = ensure(L.c, nc * sizeof(T))))
    return rc;
  // device bases: base[idx] mirrors host element idx over each full span
  const int64_t lo_a = a.off + p.fp_lo[0], lo_b = b.off + p.fp_lo[1], lo_c = off_c + p.fp_lo[2];
  T* base_a = (T*)L.a.p - lo_a;
  T* base_b = (T*)L.b.p - lo_b;
  T* base_c = (T*)L.c.p - lo_c;
  if (cut.owner == 0) CK(cudaMemcpyAsync(base_b + lo_b, hb + lo_b, nb * sizeof(T), cudaMemcpyHostToDevice, L.h2d));
  else CK(cudaMemcpyAsync(base_a + lo_a, ha + lo_a, na * sizeof(T), cudaMemcpyHostToDevice, L.h2d));
  rc = issue_slabs<T>(L, ds, cut, a, b, s, p, ha, hb, hc, off_c, len_c, 0, cut.E, S, base_a, base_b,
                      base_c, 0);
  if (rc) return rc;
  CK(cudaStreamSynchronize(L.d2h));
  CK(cudaStreamSynchronize(L.stream));
  return 0;
}

// ---------------------------------------------------------------------------
// Multi-device xGETT: one host call drives a list of devices.
//   slabs   — the slab mode (slab_cut) is split into one row range per device;
//             each device copies its slabs of the owner operand and of C over
//             its own PCIe link (pipelined, issue_slabs) and computes them; the
//             replicated operand crosses PCIe once in total: device j copies
//             chunk j of its span from the host and the devices exchange the
//             chunks over NVLink (cudaMemcpyPeerAsync).  No collective.
//   split-K — when the free extents are too small to fill the devices (c5):
//             the contracted pair with the largest extent is split, device 0
//             computes C += A_0·B_0, device j > 0 computes P_j = A_j·B_j into
//             a zeroed copy of C's span, and device 0 adds
//             C += (P_1 + ... + P_{n-1}) in that fixed order (deterministic),
//             reading the partials straight from the peers' memory over
//             NVLink (or staging them with cudaMemcpyPeerAsync when peer
//             access is unavailable) — the one reduce of the call.
// A device listed k times contributes k lanes (its lanes 0..k-1), so the
// whole path runs on a single GPU with devices = (0, 0).

std::mutex g_peer_mu;
signed char g_peer[kMaxDevices][kMaxDevices];  // 0 unknown, 1 enabled, -1 unavailable

// can device `dev` load from `peer`'s memory?  (enables access once)
bool peer_access(int dev, int peer) {
  if (dev == peer) return true;
  std::lock_guard<std::mutex> lk(g_peer_mu);
  signed char& st = g_peer[dev][peer];
  if (st == 0) {
    int can = 0;
    st = -1;
    if (cudaDeviceCanAccessPeer(&can, dev, peer) == cudaSuccess && can) {
      int cur = -1;
      cudaGetDevice(&cur);
      cudaSetDevice(dev);
      cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
      if (e == cudaSuccess || e == cudaErrorPeerAccessAlreadyEnabled) st = 1;
      cudaGetLastError();
      cudaSetDevice(cur);
    }
  }
  return st == 1;
}

struct LaneRef {
  int dev;
  Lane* L;
};

int g_multi_force = 0;  // 0 auto, 1 slabs, 2 split-K (gett_set_multi; tests)
thread_local char t_last_multi[96] = "none";

// The multi-device schedule of a validated, non-empty call on n lanes —
// host-only (no CUDA), shared by the in-call multi-device path and by
// gett_multi_schedule (the torchrun per-rank partition, shard.py).
struct MultiSched {
  int strategy = 0;  // 0 one device, 1 slabs, 2 split-K
  int n = 1;         // lanes used
  SlabCut cut;       // slabs
  int pair = -1;     // split-K: contracted pair split
  std::vector<int64_t> lo, hi;  // per lane: rows of the cut mode / range of the pair
};

MultiSched multi_schedule(const Plan& p, const View& a, const View& b, const Spec& s, int n_in,
                          int force) {
  MultiSched m;
  int n = std::min(n_in, kMaxParts + 1);
  if (n < 2 || p.c_may_alias || p.size_free == 0 || p.size_cont == 0) return m;
  const double macs = (double)p.size_free * (double)p.size_cont;
  const int64_t tiles = ((p.gm.G + 127) / 128) * ((p.gn.G + 127) / 128);
  SlabCut cut;
  const bool can_slab = slab_cut(p, a, b, s, &cut) && cut.E >= 2 &&
                        (cut.owner_disjoint || force == 1);
  int pair = -1;
  for (int k = 0; k < s.conts; ++k)
    if (a.ext[s.cont_a[k]] >= 2 && (pair < 0 || a.ext[s.cont_a[k]] > a.ext[s.cont_a[pair]])) pair = k;
  int strategy = 0;
  if (force == 1) strategy = can_slab ? 1 : 0;
  else if (force == 2) strategy = pair >= 0 ? 2 : 0;
  else if (macs >= (double)n * (1 << 27)) {
    if (can_slab && tiles >= 74 * n) strategy = 1;  // every device gets >= half a wave of tiles
    else if (pair >= 0 && p.size_cont >= 256 * n) strategy = 2;
    else if (can_slab) strategy = 1;
  }
  if (strategy == 0) return m;
  m.strategy = strategy;
  if (strategy == 1) {
    if (n > cut.E) n = (int)cut.E;
    m.cut = cut;
    // row ranges: granules of 128 rows when every device gets at least one
    const int64_t g = cut.E >= 128 * n ? 128 : 1;
    const int64_t units = (cut.E + g - 1) / g;
    for (int i = 0; i < n; ++i) {
      m.lo.push_back(std::min(cut.E, units * i / n * g));
      m.hi.push_back(i + 1 == n ? cut.E : std::min(cut.E, units * (i + 1) / n * g));
    }
  } else {
    const int64_t Ek = a.ext[s.cont_a[pair]];
    if (n > Ek) n = (int)Ek;
    m.pair = pair;
    for (int i = 0; i < n; ++i) {
      m.lo.push_back(Ek * i / n);
      m.hi.push_back(Ek * (i + 1) / n);
    }
  }
  m.n = n;
  return m;
}

// Put the span [lo, lo + n) of host buffer h at base[i] + lo on every lane:
// lane j uploads chunk j over its own PCIe link, then every lane pulls the
// other chunks from their lanes (cudaMemcpyPeerAsync over NVLink; a plain
// device copy between two lanes of one GPU), all on the lanes' h2d streams.
// Uses event index `ev` of every lane.
template <typename T>
int replicate_span(std::vector<LaneRef>& lanes, const std::vector<T*>& base, const T* h, int64_t lo,
                   size_t n_el, size_t ev) {
  const int n = (int)lanes.size();
  std::vector<size_t> cb(n + 1);
  for (int j = 0; j <= n; ++j) cb[j] = n_el * j / n;
  int rc;
  for (int j = 0; j < n; ++j) {
    CK(cudaSetDevice(lanes[j].dev));
    Lane& L = *lanes[j].L;
    CK(cudaMemcpyAsync(base[j] + lo + cb[j], h + lo + cb[j], (cb[j + 1] - cb[j]) * sizeof(T),
                       cudaMemcpyHostToDevice, L.h2d));
    cudaEvent_t e;
    if ((rc = event_at(L, ev, &e))) return rc;
    CK(cudaEventRecord(e, L.h2d));
  }
  for (int i = 0; i < n; ++i) {
    CK(cudaSetDevice(lanes[i].dev));
    Lane& L = *lanes[i].L;
    for (int j = 0; j < n; ++j) {
      if (j == i || cb[j + 1] == cb[j]) continue;
      CK(cudaStreamWaitEvent(L.h2d, lanes[j].L->events[ev], 0));
      const size_t bytes = (cb[j + 1] - cb[j]) * sizeof(T);
      T* dst = base[i] + lo + cb[j];
      const T* src = base[j] + lo + cb[j];
      if (lanes[j].dev == lanes[i].dev) CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, L.h2d));
      else CK(cudaMemcpyPeerAsync(dst, lanes[i].dev, src, lanes[j].dev, bytes, L.h2d));
    }
  }
  return 0;
}

template <typename T>
int multi_slabs(std::vector<LaneRef>& lanes, const MultiSched& m, const View& a, const View& b,
                const Spec& s, const Plan& p, const T* ha, const T* hb, T* hc, int64_t off_c,
                int64_t len_c) {
  const int n = (int)lanes.size();
  const SlabCut& cut = m.cut;
  const size_t na = (size_t)(p.fp_hi[0] - p.fp_lo[0] + 1);
  const size_t nb = (size_t)(p.fp_hi[1] - p.fp_lo[1] + 1);
  const size_t nc = (size_t)(p.fp_hi[2] - p.fp_lo[2] + 1);
  const int64_t lo_a = a.off + p.fp_lo[0], lo_b = b.off + p.fp_lo[1], lo_c = off_c + p.fp_lo[2];
  std::vector<T*> ba(n), bb(n), bc(n);
  int rc;
  for (int i = 0; i < n; ++i) {
    CK(cudaSetDevice(lanes[i].dev));
    Lane& L = *lanes[i].L;
    if ((rc = ensure(L.a, na * sizeof(T))) || (rc = ensure(L.b, nb * sizeof(T))) ||
        (rc = ensure(L.c, nc * sizeof(T))))
      return rc;
    ba[i] = (T*)L.a.p - lo_a;
    bb[i] = (T*)L.b.p - lo_b;
    bc[i] = (T*)L.c.p - lo_c;
  }
  // the replicated operand: chunk j over lane j's PCIe link, then NVLink
  if (cut.owner == 0) rc = replicate_span<T>(lanes, bb, hb, lo_b, nb, 0);
  else rc = replicate_span<T>(lanes, ba, ha, lo_a, na, 0);
  if (rc) return rc;
  // each lane's rows, pipelined over its own copy streams
  for (int i = 0; i < n; ++i) {
    const int64_t r0 = m.lo[i], r1 = m.hi[i];
    if (r1 == r0) continue;
    CK(cudaSetDevice(lanes[i].dev));
    const size_t lane_bytes = (size_t)((double)(na + 2 * nc) * (r1 - r0) / cut.E) * sizeof(T);
    int64_t S = g_pipeline_slabs > 1 ? g_pipeline_slabs : (int64_t)std::min<size_t>(10, 1 + lane_bytes / (8u << 20));
    if (g_pipeline_slabs == 0 || g_pipeline_slabs == 1) S = 1;
    if (S > r1 - r0) S = r1 - r0;
    rc = issue_slabs<T>(*lanes[i].L, g_dev[lanes[i].dev], cut, a, b, s, p, ha, hb, hc, off_c, len_c,
                        r0, r1, S, ba[i], bb[i], bc[i], 1);
    if (rc) return rc;
  }
  for (int i = 0; i < n; ++i) {
    CK(cudaSetDevice(lanes[i].dev));
    CK(cudaStreamSynchronize(lanes[i].L->d2h));
    CK(cudaStreamSynchronize(lanes[i].L->stream));
    CK(cudaStreamSynchronize(lanes[i].L->h2d));
  }
  std::snprintf(t_last_multi, sizeof t_last_multi, "slabs x%d (mode %d of %c, replicated %c over peers)", n,
                cut.dim, cut.owner == 0 ? 'A' : 'B', cut.owner == 0 ? 'B' : 'A');
  return 0;
}

template <typename T>
int multi_splitk(std::vector<LaneRef>& lanes, const MultiSched& m, const View& a, const View& b,
                 const Spec& s, const Plan& p, const T* ha, const T* hb, T* hc, int64_t off_c,
                 int64_t len_c) {
  const int n = (int)lanes.size();
  const int pair = m.pair;
  const int da = (int)s.cont_a[pair], db = (int)s.cont_b[pair];
  const size_t na = (size_t)(p.fp_hi[0] - p.fp_lo[0] + 1);
  const size_t nb = (size_t)(p.fp_hi[1] - p.fp_lo[1] + 1);
  const size_t nc = (size_t)(p.fp_hi[2] - p.fp_lo[2] + 1);
  const int64_t lo_a = a.off + p.fp_lo[0], lo_b = b.off + p.fp_lo[1], lo_c = off_c + p.fp_lo[2];
  std::vector<T*> ba(n), bb(n), bc(n);
  int rc;
  for (int i = 0; i < n; ++i) {
    CK(cudaSetDevice(lanes[i].dev));
    Lane& L = *lanes[i].L;
    if ((rc = ensure(L.a, na * sizeof(T))) || (rc = ensure(L.b, nb * sizeof(T))) ||
        (rc = ensure(L.c, nc * sizeof(T))))
      return rc;
    ba[i] = (T*)L.a.p - lo_a;
    bb[i] = (T*)L.b.p - lo_b;
    bc[i] = (T*)L.c.p - lo_c;
  }
  // A and B cross PCIe once in total (a K slice of a strided view spans
  // nearly the whole buffer: c5's A, split along any pair, still does), C
  // once to lane 0; lanes j > 0 accumulate into zeroed copies of C's span
  if ((rc = replicate_span<T>(lanes, ba, ha, lo_a, na, 0))) return rc;
  if ((rc = replicate_span<T>(lanes, bb, hb, lo_b, nb, 1))) return rc;
  for (int i = 0; i < n; ++i) {
    CK(cudaSetDevice(lanes[i].dev));
    Lane& L = *lanes[i].L;
    const int64_t k0 = m.lo[i], k1 = m.hi[i];
    std::vector<int64_t> ea(a.ext, a.ext + a.rank), eb(b.ext, b.ext + b.rank);
    ea[da] = k1 - k0;
    eb[db] = k1 - k0;
    View sa = a, sb = b;
    sa.ext = ea.data(); sa.off = a.off + k0 * a.inc[da];
    sb.ext = eb.data(); sb.off = b.off + k0 * b.inc[db];
    std::shared_ptr<DevPlan> dp;
    if ((rc = get_plan(sizeof(T) == 8 ? 'd' : 's', sa, sb, s, off_c, len_c, &dp))) return rc;
    if (i == 0) CK(cudaMemcpyAsync(L.c.p, hc + lo_c, nc * sizeof(T), cudaMemcpyHostToDevice, L.h2d));
    else CK(cudaMemsetAsync(L.c.p, 0, nc * sizeof(T), L.h2d));
    cudaEvent_t ein, e;
    if ((rc = event_at(L, 2, &ein)) || (rc = event_at(L, 3, &e))) return rc;
    CK(cudaEventRecord(ein, L.h2d));
    CK(cudaStreamWaitEvent(L.stream, ein, 0));
    if ((rc = run_device<T>(*dp, ba[i] + sa.off, bb[i] + sb.off, bc[i] + off_c, L.stream, g_dev[lanes[i].dev])))
      return rc;
    CK(cudaEventRecord(e, L.stream));
  }
  // device 0: C += (P_1 + ... + P_{n-1}), then C's span back to the host
  const int d0 = lanes[0].dev;
  Lane& L0 = *lanes[0].L;
  CK(cudaSetDevice(d0));
  bool direct = !g_multi_stage;
  for (int j = 1; j < n && direct; ++j) direct = peer_access(d0, lanes[j].dev);
  AccumParams<T> ap;
  ap.C = bc[0] + off_c;
  ap.n = n - 1;
  if (!direct && (rc = ensure(L0.red, (size_t)(n - 1) * nc * sizeof(T)))) return rc;
  for (int j = 1; j < n; ++j) {
    CK(cudaStreamWaitEvent(L0.stream, lanes[j].L->events[3], 0));
    if (direct) {
      ap.P[j - 1] = bc[j] + off_c;
    } else {
      T* dst = (T*)L0.red.p + (size_t)(j - 1) * nc;
      if (lanes[j].dev == d0)
        CK(cudaMemcpyAsync(dst, lanes[j].L->c.p, nc * sizeof(T), cudaMemcpyDeviceToDevice, L0.stream));
      else
        CK(cudaMemcpyPeerAsync(dst, d0, lanes[j].L->c.p, lanes[j].dev, nc * sizeof(T), L0.stream));
      ap.P[j - 1] = dst - lo_c + off_c;
    }
  }
  std::shared_ptr<DevPlan> vp;
  if ((rc = get_view_plan(p.rank_c, p.ext_c.data(), s.inc_c, &vp))) return rc;
  ap.g = vp->gm;
  CK(launch_accum<T>(ap, L0.stream));
  ++g_launches;
  CK(cudaMemcpyAsync(hc + lo_c, L0.c.p, nc * sizeof(T), cudaMemcpyDeviceToHost, L0.stream));
  CK(cudaStreamSynchronize(L0.stream));
  for (int j = 1; j < n; ++j) {
    CK(cudaSetDevice(lanes[j].dev));
    CK(cudaStreamSynchronize(lanes[j].L->stream));
    CK(cudaStreamSynchronize(lanes[j].L->h2d));
  }
  std::snprintf(t_last_multi, sizeof t_last_multi, "split-K x%d (pair %d, %s reduce)", n, pair,
                direct ? "peer-load" : "staged");
  return 0;
}

// Choose the multi-device strategy of a validated, non-empty host call.
// Returns kNotPipelined when the call should run on devices[0] alone.
template <typename T>
int host_multi(const Plan& p, const View& a, const View& b, const Spec& s, const T* ha,
               const T* hb, T* hc, int64_t off_c, int64_t len_c, const std::vector<int>& devs) {
  const MultiSched m = multi_schedule(p, a, b, s, (int)devs.size(), g_multi_force);
  if (m.strategy == 0) return kNotPipelined;
  const int n = m.n;
  // lock the distinct devices in ascending order, then take lanes
  std::vector<int> order(devs.begin(), devs.begin() + n);
  std::sort(order.begin(), order.end());
  order.erase(std::unique(order.begin(), order.end()), order.end());
  std::vector<std::unique_lock<std::mutex>> locks;
  for (int d : order) locks.emplace_back(g_dev[d].mu);
  std::vector<LaneRef> lanes(n);
  std::vector<int> used(kMaxDevices, 0);
  int rc;
  for (int i = 0; i < n; ++i) {
    CK(cudaSetDevice(devs[i]));
    lanes[i].dev = devs[i];
    if ((rc = get_lane(devs[i], (size_t)used[devs[i]]++, &lanes[i].L))) return rc;
  }
  return m.strategy == 1 ? multi_slabs<T>(lanes, m, a, b, s, p, ha, hb, hc, off_c, len_c)
                         : multi_splitk<T>(lanes, m, a, b, s, p, ha, hb, hc, off_c, len_c);
}

int fill_errors(const std::vector<Error>& errs, int32_t* codes, int64_t* info, int max_errs) {
  int n = (int)errs.size();
  for (int i = 0; i < n && i < max_errs; ++i) {
    if (codes) codes[i] = errs[i].code;
    if (info)
      for (int w = 0; w < GETT_ERR_INFO_WORDS; ++w) info[i * GETT_ERR_INFO_WORDS + w] = errs[i].info[w];
  }
  return n;
}

// marks the calling thread's device call as captured (plans it touches are
// pinned) for the duration of one entry point
struct CaptureScope {
  explicit CaptureScope(cudaStream_t s) {
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    t_capturing = cudaStreamIsCapturing(s, &st) == cudaSuccess && st != cudaStreamCaptureStatusNone;
  }
  ~CaptureScope() { t_capturing = false; }
};

// devices of a host call: explicit list, else the gett_set_devices default,
// else none (the current device)
int check_devices(int n_dev, const int32_t* devices, std::vector<int>* out) {
  out->clear();
  if (n_dev > 0) {
    if (!devices) {
      t_last_error = "devices is NULL";
      return GETT_E_INVALID_ARG;
    }
    for (int i = 0; i < n_dev; ++i) {
      if (devices[i] < 0 || devices[i] >= kMaxDevices) {
        t_last_error = "device ordinal out of range";
        return GETT_E_INVALID_ARG;
      }
      out->push_back(devices[i]);
    }
  } else {
    std::lock_guard<std::mutex> lk(g_plan_mu);
    *out = g_devices;
  }
  return 0;
}

// Run a validated, non-empty call on its plan (gett_impl after validation,
// and gett_execute on a plan handle): multi-device host calls, else the
// current device's lane 0 — device pointers stream-ordered, host buffers
// through the (pipelined) copy path.
template <typename T>
int execute_plan(bool host, DevPlan& dpr, const View& va, const View& vb, const Spec& sp, const T* a,
                 const T* b, T* c, int64_t off_a, int64_t off_b, int64_t off_c, int64_t len_c,
                 cudaStream_t stream, const std::vector<int>& devs) {
  int rc = 0;
  const Plan& p = dpr.plan;
  if (host && devs.size() > 1) {
    for (int d : devs) {
      cudaError_t e = cudaSetDevice(d);
      if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice(devices[i])");
    }
    rc = host_multi<T>(p, va, vb, sp, a, b, c, off_c, len_c, devs);
    if (rc != kNotPipelined) return rc;
    CK(cudaSetDevice(devs[0]));
  }
  int dev;
  if ((rc = current_device(&dev))) return rc;
  DevState& ds = g_dev[dev];
  std::lock_guard<std::mutex> lk(ds.mu);
  if (!host) {
    CaptureScope cs(stream);
    if (t_capturing) dpr.pinned = true;
    return run_device<T>(dpr, a + off_a, b + off_b, c + off_c, stream, ds);
  }
  Lane* Lp = nullptr;
  if ((rc = get_lane(dev, 0, &Lp))) return rc;
  Lane& L = *Lp;
  rc = host_pipelined<T>(dpr, va, vb, sp, a, b, c, off_c, len_c, ds, L);
  if (rc != kNotPipelined) return rc;
  // host buffers: copy the addressed spans in, run, copy C's span back
  // (the plan is cached by descriptor only: spans use this call's offsets)
  const int64_t lo_a = off_a + p.fp_lo[0], lo_b = off_b + p.fp_lo[1], lo_c = off_c + p.fp_lo[2];
  size_t na = (size_t)(p.fp_hi[0] - p.fp_lo[0] + 1);
  size_t nb = (size_t)(p.fp_hi[1] - p.fp_lo[1] + 1);
  size_t nc = (size_t)(p.fp_hi[2] - p.fp_lo[2] + 1);
  if ((rc = ensure(L.a, na * sizeof(T))) || (rc = ensure(L.b, nb * sizeof(T))) ||
      (rc = ensure(L.c, nc * sizeof(T))))
    return rc;
  T* da = (T*)L.a.p;
  T* db = (T*)L.b.p;
  T* dc = (T*)L.c.p;
  cudaStream_t s = L.stream;
  CK(cudaMemcpyAsync(da, a + lo_a, na * sizeof(T), cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(db, b + lo_b, nb * sizeof(T), cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(dc, c + lo_c, nc * sizeof(T), cudaMemcpyHostToDevice, s));
  rc = run_device<T>(dpr, da - p.fp_lo[0], db - p.fp_lo[1], dc - p.fp_lo[2], s, ds);
  if (rc) return rc;
  CK(cudaMemcpyAsync(c + lo_c, dc, nc * sizeof(T), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return 0;
}

template <typename T>
int gett_impl(bool host, int rank_a, const int64_t* ext_a, const int64_t* inc_a, const T* a,
              int64_t off_a, int64_t len_a, int rank_b, const int64_t* ext_b,
              const int64_t* inc_b, const T* b, int64_t off_b, int64_t len_b, int conts,
              const int64_t* cont_a, const int64_t* cont_b, int perm_len, const int64_t* perm,
              int inc_c_len, const int64_t* inc_c, T* c, int64_t off_c, int64_t len_c,
              cudaStream_t stream, int32_t* codes, int64_t* info, int max_errs, int n_dev = 0,
              const int32_t* devices = nullptr) {
  if (rank_a < 0 || rank_b < 0 || conts < 0 || perm_len < 0 || inc_c_len < 0 || off_a < 0 ||
      off_b < 0 || off_c < 0 || len_a < 0 || len_b < 0 || len_c < 0 || n_dev < 0) {
    t_last_error = "negative rank/count/offset/length";
    return GETT_E_INVALID_ARG;
  }
  read_env();
  t_last_kernel = "none";
  std::snprintf(t_last_multi, sizeof t_last_multi, "none");
  std::vector<int> devs;
  int rc = 0;
  if (host && (rc = check_devices(n_dev, devices, &devs))) return rc;
  DeviceGuard guard;  // a call on devices[0] / several devices restores the caller's device
  // (validation needs no device: a bad ordinal is reported after it)
  cudaError_t set_err = devs.empty() ? cudaSuccess : cudaSetDevice(devs[0]);
  if (set_err != cudaSuccess) cudaGetLastError();
  View va{rank_a, ext_a, inc_a, off_a, len_a};
  View vb{rank_b, ext_b, inc_b, off_b, len_b};
  Spec sp{conts, cont_a, cont_b, perm_len, perm, inc_c_len, inc_c};
  View vc{0, nullptr, nullptr, off_c, len_c};
  // a call whose descriptor (every argument but the pointers) equals the last
  // validated one reuses its result and plan: no validation or plan-key work
  // (validation runs without CUDA: the device is only queried on a key match)
  std::vector<int64_t>& key = t_key;
  key.clear();
  key.push_back((int64_t)sizeof(T));
  auto put = [&](int n, const int64_t* v) {
    key.push_back(n);
    for (int i = 0; i < n; ++i) key.push_back(v[i]);
  };
  put(rank_a, ext_a); put(rank_a, inc_a); key.push_back(off_a); key.push_back(len_a);
  put(rank_b, ext_b); put(rank_b, inc_b); key.push_back(off_b); key.push_back(len_b);
  put(conts, cont_a); put(conts, cont_b); put(perm_len, perm); put(inc_c_len, inc_c);
  key.push_back(off_c); key.push_back(len_c);
  std::shared_ptr<DevPlan> dp;
  {
    std::lock_guard<std::mutex> lk(g_plan_mu);
    int cur_dev = -1;
    if (g_last.dp && key == g_last.key && cudaGetDevice(&cur_dev) == cudaSuccess &&
        cur_dev == g_last.dp->device)
      dp = g_last.dp;
  }
  if (!dp) {
    std::vector<Error> errs = validate(va, vb, sp, CMode::Derived, vc);
    if (!errs.empty()) return fill_errors(errs, codes, info, max_errs);
    // empty iteration space: nothing is written (kernel.py:93-94)
    for (int d = 0; d < rank_a; ++d)
      if (ext_a[d] == 0) return 0;
    for (int d = 0; d < rank_b; ++d)
      if (ext_b[d] == 0) return 0;
    if ((rc = get_plan(sizeof(T) == 8 ? 'd' : 's', va, vb, sp, off_c, len_c, &dp))) return rc;
    std::lock_guard<std::mutex> lk(g_plan_mu);
    g_last.key = key;
    g_last.dp = dp;
  }
  if (set_err != cudaSuccess) return cuda_fail(set_err, "cudaSetDevice(devices[0])");
  return execute_plan<T>(host, *dp, va, vb, sp, a, b, c, off_a, off_b, off_c, len_c, stream, devs);
}

// Complex contraction as ONE real GETT on a real embedding.  The operand with
// fewer elements (X; the other is Y) is expanded into a dense workspace X'
// with two extra modes: q (contracted against a new stride-1 re/im mode of Y)
// and s (a new stride-1 re/im mode of C):
//   X'[.., q=0, .., s] = (re x, im x),   X'[.., q=1, .., s] = (-im x, re x)
// so  C[.., s] += sum_{k,q} Y[k, q] X'[k, q, .., s]  is the complex product
// (re c += re y re x - im y im x,  im c += re y im x + im y re x).  X' puts s
// first, then X's free modes in C's stride order, then q, then the contracted
// modes in Y's stride order, so the new modes fold into the neighbouring
// groups (an M x 2N x 2K real GETT with the same inner strides as a real call).
template <typename R>
int run_complex_embedded(const View& va, const View& vb, const Spec& sp, const R* a2, const R* b2,
                         R* c2, cudaStream_t stream, DevState& ds) {
  auto count = [](const View& v) {
    int64_t n = 1;
    for (int d = 0; d < v.rank; ++d) n *= v.ext[d];
    return n;
  };
  const bool swap = count(va) < count(vb);  // expand A (operand order Y = B, X = A)
  const View& vy = swap ? vb : va;
  const View& vx = swap ? va : vb;
  const int64_t* cy = swap ? sp.cont_b : sp.cont_a;
  const int64_t* cx = swap ? sp.cont_a : sp.cont_b;
  const R* py = swap ? b2 : a2;
  const R* px = swap ? a2 : b2;
  // old free-list index of every free mode (A's free modes, then B's)
  auto free_index = [&](const View& v, const int64_t* cont, int base, std::vector<int>& out) {
    out.assign(v.rank, -1);
    for (int d = 0; d < v.rank; ++d) {
      bool c = false;
      for (int j = 0; j < sp.conts; ++j) c |= cont[j] == d;
      if (!c) out[d] = base++;
    }
    return base;
  };
  std::vector<int> fa, fb;
  const int nfa = free_index(va, sp.cont_a, 0, fa);
  free_index(vb, sp.cont_b, nfa, fb);
  const std::vector<int>& fy = swap ? fb : fa;
  const std::vector<int>& fx = swap ? fa : fb;
  // X' strides (real elements): s = 1, free modes by |C stride|, q, contracted by |Y stride|
  std::vector<int> xfree, xcont(sp.conts);
  for (int d = 0; d < vx.rank; ++d)
    if (fx[d] >= 0) xfree.push_back(d);
  std::stable_sort(xfree.begin(), xfree.end(), [&](int x, int y) {
    return std::llabs(sp.inc_c[sp.perm[fx[x]]]) < std::llabs(sp.inc_c[sp.perm[fx[y]]]);
  });
  for (int j = 0; j < sp.conts; ++j) xcont[j] = j;
  std::stable_sort(xcont.begin(), xcont.end(), [&](int x, int y) {
    return std::llabs(vy.inc[cy[x]]) < std::llabs(vy.inc[cy[y]]);
  });
  ExpandParams<R> ep{};
  std::vector<int64_t> xinc(vx.rank + 2);
  int64_t st = 2;
  ep.n = 0;
  for (int d : xfree) {
    xinc[d] = st;
    ep.ext[ep.n] = vx.ext[d]; ep.inc[ep.n] = vx.inc[d]; ep.dst_st[ep.n] = st; ++ep.n;
    st *= vx.ext[d];
  }
  const int64_t q = st;
  st *= 2;
  for (int j : xcont) {
    const int d = (int)cx[j];
    xinc[d] = st;
    ep.ext[ep.n] = vx.ext[d]; ep.inc[ep.n] = vx.inc[d]; ep.dst_st[ep.n] = st; ++ep.n;
    st *= vx.ext[d];
  }
  xinc[vx.rank] = q;
  xinc[vx.rank + 1] = 1;
  ep.total = 1;
  for (int i = 0; i < ep.n; ++i) ep.total *= ep.ext[i];
  ep.q = q;
  ep.src = px;
  StreamWs& sw = ds.sws[stream];
  int rc = ensure(sw.cx, (size_t)st * sizeof(R));
  if (rc) return rc;
  ep.dst = (R*)sw.cx.p;
  CK(launch_expand_complex<R>(ep, stream));
  ++g_launches;
  // the real spec: Y' = Y + (re/im, stride 1), X' as laid out above, C + (s, stride 1)
  std::vector<int64_t> yext(vy.ext, vy.ext + vy.rank), yinc(vy.rank + 1), xext(vx.ext, vx.ext + vx.rank);
  for (int d = 0; d < vy.rank; ++d) yinc[d] = 2 * vy.inc[d];
  yext.push_back(2);
  yinc[vy.rank] = 1;
  xext.push_back(2);
  xext.push_back(2);
  std::vector<int64_t> cy2(cy, cy + sp.conts), cx2(cx, cx + sp.conts);
  cy2.push_back(vy.rank);
  cx2.push_back(vx.rank);
  std::vector<int64_t> perm2, inc_c2(sp.inc_c_len + 1);
  for (int d = 0; d < vy.rank; ++d)
    if (fy[d] >= 0) perm2.push_back(sp.perm[fy[d]]);
  for (int d = 0; d < vx.rank; ++d)
    if (fx[d] >= 0) perm2.push_back(sp.perm[fx[d]]);
  perm2.push_back(sp.inc_c_len);
  for (int d = 0; d < sp.inc_c_len; ++d) inc_c2[d] = 2 * sp.inc_c[d];
  inc_c2[sp.inc_c_len] = 1;
  View ry{vy.rank + 1, yext.data(), yinc.data(), 0, 2 * vy.len};
  View rx{vx.rank + 2, xext.data(), xinc.data(), 0, st};
  Spec rs{sp.conts + 1, cy2.data(), cx2.data(), (int)perm2.size(), perm2.data(), sp.inc_c_len + 1, inc_c2.data()};
  std::shared_ptr<DevPlan> rp;
  if ((rc = get_plan(sizeof(R) == 8 ? 'd' : 's', ry, rx, rs, 0, 0, &rp))) return rc;
  if ((rc = run_device<R>(*rp, py, ep.dst, c2, stream, ds, 0, true))) return rc;
  t_last_kernel = sizeof(R) == 8 ? "zgett_embedded_dmma" : "cgett_embedded_tc3xtf32";
  return 0;
}

// Complex contraction on device buffers.  a2/b2/c2 point at each view's base
// element as a real (re, im)-interleaved array.  ref/serial: complex kernels
// in reference order; tiled: four real GETTs on the re/im sub-views (every
// increment doubled; im = base + 1) through the tensor-core kernels:
//   C.re += A.re B.re,  C.re -= A.im B.im,  C.im += A.re B.im,  C.im += A.im B.re
template <typename R>
int run_complex(DevPlan& cp, const View& va, const View& vb, const Spec& sp, const R* a2,
                const R* b2, R* c2, cudaStream_t stream, DevState& ds) {
  const Plan& p = cp.plan;
  Mode mode = g_mode;
  if (p.c_may_alias) mode = Mode::Serial;
  const int64_t M = p.gm.G, N = p.gn.G, K = p.gk.G;
  if (mode == Mode::Auto) mode = (K <= 8 || M * N * K <= (1LL << 18)) ? Mode::Ref : Mode::Tiled;
  const bool z = sizeof(R) == 8;
  if (mode == Mode::Serial) {
    SerialParams<R> s;
    s.A = a2; s.B = b2; s.C = c2;
    s.num_free = cp.serial_nf;
    s.num_cont = cp.serial_nc;
    s.size_free = p.size_free;
    s.size_cont = p.size_cont;
    s.tab = cp.serial_tab;
    warn_serial(p.size_free, p.size_cont);
    CK(launch_serial_c<R>(s, stream));
    ++g_launches;
    t_last_kernel = z ? "zgett_serial" : "cgett_serial";
    return 0;
  }
  if (mode == Mode::Ref) {
    RefParams<R> rp;
    rp.A = p.swapped ? b2 : a2;
    rp.B = p.swapped ? a2 : b2;
    rp.C = c2;
    rp.gm = cp.gm; rp.gn = cp.gn;
    rp.M = (int32_t)M; rp.N = (int32_t)N;
    rp.k_inner = (int32_t)p.gk_ref.e_in;
    rp.k_sa = p.gk_ref.s_in[0];
    rp.k_sb = p.gk_ref.s_in[1];
    rp.k_outer = (int32_t)p.gk_ref.T[0].size();
    rp.kta = cp.kref_a;
    rp.ktb = cp.kref_b;
    CK(launch_ref_c<R>(rp, stream));
    ++g_launches;
    t_last_kernel = z ? "zgett_ref_order" : "cgett_ref_order";
    return 0;
  }
  if (std::max(va.rank, vb.rank) + 2 <= kExpandMaxModes && !g_complex_4x)
    return run_complex_embedded<R>(va, vb, sp, a2, b2, c2, stream, ds);
  // real sub-views: same extents, doubled increments
  std::vector<int64_t> ia(va.rank), ib(vb.rank), ic(sp.inc_c_len);
  for (int d = 0; d < va.rank; ++d) ia[d] = 2 * va.inc[d];
  for (int d = 0; d < vb.rank; ++d) ib[d] = 2 * vb.inc[d];
  for (int d = 0; d < sp.inc_c_len; ++d) ic[d] = 2 * sp.inc_c[d];
  View ra{va.rank, va.ext, ia.data(), 0, 2 * va.len};
  View rb{vb.rank, vb.ext, ib.data(), 0, 2 * vb.len};
  Spec rs = sp;
  rs.inc_c = ic.data();
  std::shared_ptr<DevPlan> rp;
  int rc = get_plan(z ? 'd' : 's', ra, rb, rs, 0, 0, &rp);
  if (rc) return rc;
  if ((rc = run_device<R>(*rp, a2, b2, c2, stream, ds, 0, true))) return rc;
  if ((rc = run_device<R>(*rp, a2 + 1, b2 + 1, c2, stream, ds, 1, true))) return rc;
  if ((rc = run_device<R>(*rp, a2, b2 + 1, c2 + 1, stream, ds, 0, true))) return rc;
  if ((rc = run_device<R>(*rp, a2 + 1, b2, c2 + 1, stream, ds, 0, true))) return rc;
  t_last_kernel = z ? "zgett_4x_dmma" : "cgett_4x_tc3xtf32";
  return 0;
}

// cgett / zgett: pointers are interleaved (re, im) reals; offsets, lengths and
// increments count complex elements (the reference's complex64/128 buffers).
template <typename R>
int gett_impl_complex(bool host, int rank_a, const int64_t* ext_a, const int64_t* inc_a,
                      const R* a, int64_t off_a, int64_t len_a, int rank_b, const int64_t* ext_b,
                      const int64_t* inc_b, const R* b, int64_t off_b, int64_t len_b, int conts,
                      const int64_t* cont_a, const int64_t* cont_b, int perm_len,
                      const int64_t* perm, int inc_c_len, const int64_t* inc_c, R* c,
                      int64_t off_c, int64_t len_c, cudaStream_t stream, int32_t* codes,
                      int64_t* info, int max_errs) {
  if (rank_a < 0 || rank_b < 0 || conts < 0 || perm_len < 0 || inc_c_len < 0 || off_a < 0 ||
      off_b < 0 || off_c < 0 || len_a < 0 || len_b < 0 || len_c < 0) {
    t_last_error = "negative rank/count/offset/length";
    return GETT_E_INVALID_ARG;
  }
  read_env();
  t_last_kernel = "none";
  View va{rank_a, ext_a, inc_a, off_a, len_a};
  View vb{rank_b, ext_b, inc_b, off_b, len_b};
  Spec sp{conts, cont_a, cont_b, perm_len, perm, inc_c_len, inc_c};
  View vc{0, nullptr, nullptr, off_c, len_c};
  std::vector<Error> errs = validate(va, vb, sp, CMode::Derived, vc);
  if (!errs.empty()) return fill_errors(errs, codes, info, max_errs);
  for (int d = 0; d < rank_a; ++d)
    if (ext_a[d] == 0) return 0;
  for (int d = 0; d < rank_b; ++d)
    if (ext_b[d] == 0) return 0;
  std::shared_ptr<DevPlan> cp;
  int rc = get_plan(sizeof(R) == 8 ? 'z' : 'c', va, vb, sp, off_c, len_c, &cp);
  if (rc) return rc;
  const Plan& p = cp->plan;
  int dev;
  if ((rc = current_device(&dev))) return rc;
  DevState& ds = g_dev[dev];
  std::lock_guard<std::mutex> lk(ds.mu);
  Lane* Lp = nullptr;
  if ((rc = get_lane(dev, 0, &Lp))) return rc;
  Lane& L = *Lp;
  if (!host) {
    CaptureScope cs(stream);
    if (t_capturing) cp->pinned = true;
    return run_complex<R>(*cp, va, vb, sp, a + 2 * off_a, b + 2 * off_b, c + 2 * off_c, stream, ds);
  }
  const int64_t lo_a = off_a + p.fp_lo[0], lo_b = off_b + p.fp_lo[1], lo_c = off_c + p.fp_lo[2];
  const size_t na = (size_t)(p.fp_hi[0] - p.fp_lo[0] + 1) * 2;
  const size_t nb = (size_t)(p.fp_hi[1] - p.fp_lo[1] + 1) * 2;
  const size_t nc = (size_t)(p.fp_hi[2] - p.fp_lo[2] + 1) * 2;
  if ((rc = ensure(L.a, na * sizeof(R))) || (rc = ensure(L.b, nb * sizeof(R))) ||
      (rc = ensure(L.c, nc * sizeof(R))))
    return rc;
  R* da = (R*)L.a.p;
  R* db = (R*)L.b.p;
  R* dc = (R*)L.c.p;
  cudaStream_t s = L.stream;
  CK(cudaMemcpyAsync(da, a + 2 * lo_a, na * sizeof(R), cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(db, b + 2 * lo_b, nb * sizeof(R), cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(dc, c + 2 * lo_c, nc * sizeof(R), cudaMemcpyHostToDevice, s));
  rc = run_complex<R>(*cp, va, vb, sp, da - 2 * p.fp_lo[0], db - 2 * p.fp_lo[1], dc - 2 * p.fp_lo[2], s, ds);
  if (rc) return rc;
  CK(cudaMemcpyAsync(c + 2 * lo_c, dc, nc * sizeof(R), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return 0;
}

template <typename T>
int zero_impl(bool host, int rank, const int64_t* ext, const int64_t* inc, int64_t off,
              int64_t len, T* buf, cudaStream_t stream) {
  if (rank < 0 || rank > 64 || off < 0 || len < 0) {
    t_last_error = "bad zero_view descriptor";
    return GETT_E_INVALID_ARG;
  }
  // view_offsets (layout.py:128-140) addresses nothing when an extent is
  // zero, and nothing when one is negative (np.arange of a negative count)
  for (int d = 0; d < rank; ++d)
    if (ext[d] <= 0) return 0;
  int64_t lo, hi;
  footprint(rank, ext, inc, &lo, &hi);
  if (off + lo < 0 || off + hi >= len) {
    t_last_error = "view footprint outside the buffer";
    return GETT_E_INVALID_ARG;
  }
  std::shared_ptr<DevPlan> dp;
  int rc = get_view_plan(rank, ext, inc, &dp);
  if (rc) return rc;
  int dev;
  if ((rc = current_device(&dev))) return rc;
  DevState& ds = g_dev[dev];
  std::lock_guard<std::mutex> lk(ds.mu);
  Lane* Lp = nullptr;
  if ((rc = get_lane(dev, 0, &Lp))) return rc;
  Lane& L = *Lp;
  if (!host) {
    CK(launch_zero<T>(buf + off, dp->gm, stream));
    ++g_launches;
    return 0;
  }
  size_t n = (size_t)(hi - lo + 1);
  if ((rc = ensure(L.c, n * sizeof(T)))) return rc;
  T* d = (T*)L.c.p;
  cudaStream_t s = L.stream;
  CK(cudaMemcpyAsync(d, buf + off + lo, n * sizeof(T), cudaMemcpyHostToDevice, s));
  CK(launch_zero<T>(d - lo, dp->gm, s));
  ++g_launches;
  CK(cudaMemcpyAsync(buf + off + lo, d, n * sizeof(T), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return 0;
}

// pack: the view's addressed elements in canonical order (dimension 0
// fastest).  Host form: H2D of the view's span, gather, D2H of the n packed
// elements.
int pack_impl(bool host, int rank, const int64_t* ext, const int64_t* inc, int64_t off, int64_t len,
              int elem_bytes, const void* src, void* dst, cudaStream_t stream) {
  if (rank < 0 || rank > kPackMaxRank || off < 0 || len < 0 ||
      (elem_bytes != 4 && elem_bytes != 8 && elem_bytes != 16) || (rank > 0 && (!ext || !inc))) {
    t_last_error = "bad pack descriptor (rank <= 32, element of 4, 8 or 16 bytes)";
    return GETT_E_INVALID_ARG;
  }
  int64_t n = 1;
  for (int d = 0; d < rank; ++d) {
    if (ext[d] < 0) {
      t_last_error = "negative extent";
      return GETT_E_INVALID_ARG;
    }
    n *= ext[d];
  }
  if (n == 0) return 0;
  int64_t lo, hi;
  footprint(rank, ext, inc, &lo, &hi);
  if (off + lo < 0 || off + hi >= len) {
    t_last_error = "view footprint outside the buffer";
    return GETT_E_INVALID_ARG;
  }
  PackParams pp{};
  pp.rank = rank;
  pp.n = n;
  for (int d = 0; d < rank; ++d) {
    pp.ext[d] = ext[d];
    pp.inc[d] = inc[d];
    if (n < (1LL << 31)) pp.div[d] = FastDiv::make((int32_t)ext[d]);
  }
  int dev, rc;
  if ((rc = current_device(&dev))) return rc;
  DevState& ds = g_dev[dev];
  std::lock_guard<std::mutex> lk(ds.mu);
  const char* s8 = static_cast<const char*>(src);
  if (!host) {
    pp.src = s8 + off * elem_bytes;
    pp.dst = dst;
    CK(launch_pack(pp, elem_bytes, stream));
    ++g_launches;
    return 0;
  }
  Lane* Lp = nullptr;
  if ((rc = get_lane(dev, 0, &Lp))) return rc;
  Lane& L = *Lp;
  const size_t span = (size_t)(hi - lo + 1) * elem_bytes, out = (size_t)n * elem_bytes;
  if ((rc = ensure(L.a, span)) || (rc = ensure(L.c, out))) return rc;
  CK(cudaMemcpyAsync(L.a.p, s8 + (off + lo) * elem_bytes, span, cudaMemcpyHostToDevice, L.stream));
  pp.src = static_cast<const char*>(L.a.p) - lo * elem_bytes;
  pp.dst = L.c.p;
  CK(launch_pack(pp, elem_bytes, L.stream));
  ++g_launches;
  CK(cudaMemcpyAsync(dst, L.c.p, out, cudaMemcpyDeviceToHost, L.stream));
  CK(cudaStreamSynchronize(L.stream));
  return 0;
}

}  // namespace
}  // namespace gett

// A validated, planned call (gett_plan_create): the descriptor, its device
// plan and the device it lives on; gett_execute* skip validation, the
// descriptor key and plan lookup.
struct gett_plan_s {
  char dtype = 'd';
  bool empty = false;  // empty iteration space: executing writes nothing
  int device = 0;
  std::vector<int64_t> ext_a, inc_a, ext_b, inc_b, cont_a, cont_b, perm, inc_c;
  int64_t off_a = 0, off_b = 0, off_c = 0, len_a = 0, len_b = 0, len_c = 0;
  std::vector<int> devs;
  std::shared_ptr<gett::DevPlan> dp;
  gett::View va() const { return gett::View{(int)ext_a.size(), ext_a.data(), inc_a.data(), off_a, len_a}; }
  gett::View vb() const { return gett::View{(int)ext_b.size(), ext_b.data(), inc_b.data(), off_b, len_b}; }
  gett::Spec sp() const {
    return gett::Spec{(int)cont_a.size(), cont_a.data(), cont_b.data(), (int)perm.size(), perm.data(),
                      (int)inc_c.size(), inc_c.data()};
  }
};

namespace gett {
namespace {
template <typename T>
int execute_handle(gett_plan_s* h, bool host, const void* a, const void* b, void* c, cudaStream_t stream) {
  read_env();
  t_last_kernel = "none";
  std::snprintf(t_last_multi, sizeof t_last_multi, "none");
  if (h->empty) return 0;
  int cur = -1;
  CK(cudaGetDevice(&cur));
  if (cur != h->device) CK(cudaSetDevice(h->device));
  const View va = h->va(), vb = h->vb();
  const Spec sp = h->sp();
  static const std::vector<int> none;
  const int rc = execute_plan<T>(host, *h->dp, va, vb, sp, static_cast<const T*>(a), static_cast<const T*>(b),
                                 static_cast<T*>(c), h->off_a, h->off_b, h->off_c, h->len_c, stream,
                                 host ? h->devs : none);
  if (cur != h->device) cudaSetDevice(cur);
  return rc;
}
}  // namespace
}  // namespace gett

using namespace gett;

extern "C" {

int gett_dgett(int rank_a, const int64_t* ext_a, const int64_t* inc_a, const double* a,
               int64_t offset_a, int64_t len_a, int rank_b, const int64_t* ext_b,
               const int64_t* inc_b, const double* b, int64_t offset_b, int64_t len_b, int conts,
               const int64_t* cont_a, const int64_t* cont_b, int perm_len, const int64_t* perm,
               int inc_c_len, const int64_t* inc_c, double* c, int64_t offset_c, int64_t len_c,
               int32_t* err_codes, int64_t* err_info, int max_errs) {
  return gett_impl<double>(true, rank_a, ext_a, inc_a, a, offset_a, len_a, rank_b, ext_b, inc_b, b,
                           offset_b, len_b, conts, cont_a, cont_b, perm_len, perm, inc_c_len,
                           inc_c, c, offset_c, len_c, nullptr, err_codes, err_info, max_errs);
}

int gett_sgett(int rank_a, const int64_t* ext_a, const int64_t* inc_a, const float* a,
               int64_t offset_a, int64_t len_a, int rank_b, const int64_t* ext_b,
               const int64_t* inc_b, const float* b, int64_t offset_b, int64_t len_b, int conts,
               const int64_t* cont_a, const int64_t* cont_b, int perm_len, const int64_t* perm,
               int inc_c_len, const int64_t* inc_c, float* c, int64_t offset_c, int64_t len_c,
               int32_t* err_codes, int64_t* err_info, int max_errs) {
  return gett_impl<float>(true, rank_a, ext_a, inc_a, a, offset_a, len_a, rank_b, ext_b, inc_b, b,
                          offset_b, len_b, conts, cont_a, cont_b, perm_len, perm, inc_c_len, inc_c,
                          c, offset_c, len_c, nullptr, err_codes, err_info, max_errs);
}

int gett_dgett_device(int rank_a, const int64_t* ext_a, const int64_t* inc_a, const double* a,
                      int64_t offset_a, int64_t len_a, int rank_b, const int64_t* ext_b,
                      const int64_t* inc_b, const double* b, int64_t offset_b, int64_t len_b,
                      int conts, const int64_t* cont_a, const int64_t* cont_b, int perm_len,
                      const int64_t* perm, int inc_c_len, const int64_t* inc_c, double* c,
                      int64_t offset_c, int64_t len_c, void* stream, int32_t* err_codes,
                      int64_t* err_info, int max_errs) {
  return gett_impl<double>(false, rank_a, ext_a, inc_a, a, offset_a, len_a, rank_b, ext_b, inc_b,
                           b, offset_b, len_b, conts, cont_a, cont_b, perm_len, perm, inc_c_len,
                           inc_c, c, offset_c, len_c, (cudaStream_t)stream, err_codes, err_info,
                           max_errs);
}

int gett_sgett_device(int rank_a, const int64_t* ext_a, const int64_t* inc_a, const float* a,
                      int64_t offset_a, int64_t len_a, int rank_b, const int64_t* ext_b,
                      const int64_t* inc_b, const float* b, int64_t offset_b, int64_t len_b,
                      int conts, const int64_t* cont_a, const int64_t* cont_b, int perm_len,
                      const int64_t* perm, int inc_c_len, const int64_t* inc_c, float* c,
                      int64_t offset_c, int64_t len_c, void* stream, int32_t* err_codes,
                      int64_t* err_info, int max_errs) {
  return gett_impl<float>(false, rank_a, ext_a, inc_a, a, offset_a, len_a, rank_b, ext_b, inc_b, b,
                          offset_b, len_b, conts, cont_a, cont_b, perm_len, perm, inc_c_len, inc_c,
                          c, offset_c, len_c, (cudaStream_t)stream, err_codes, err_info, max_errs);
}

int gett_dgett_multi(int rank_a, const int64_t* ext_a, const int64_t* inc_a, const double* a,
                     int64_t offset_a, int64_t len_a, int rank_b, const int64_t* ext_b,
                     const int64_t* inc_b, const double* b, int64_t offset_b, int64_t len_b,
                     int conts, const int64_t* cont_a, const int64_t* cont_b, int perm_len,
                     const int64_t* perm, int inc_c_len, const int64_t* inc_c, double* c,
                     int64_t offset_c, int64_t len_c, int n_dev, const int32_t* devices,
                     int32_t* err_codes, int64_t* err_info, int max_errs) {
  if (n_dev < 1) {
    t_last_error = "n_dev < 1";
    return GETT_E_INVALID_ARG;
  }
  return gett_impl<double>(true, rank_a, ext_a, inc_a, a, offset_a, len_a, rank_b, ext_b, inc_b, b,
                           offset_b, len_b, conts, cont_a, cont_b, perm_len, perm, inc_c_len,
                           inc_c, c, offset_c, len_c, nullptr, err_codes, err_info, max_errs, n_dev,
                           devices);
}

int gett_sgett_multi(int rank_a, const int64_t* ext_a, const int64_t* inc_a, const float* a,
                     int64_t offset_a, int64_t len_a, int rank_b, const int64_t* ext_b,
                     const int64_t* inc_b, const float* b, int64_t offset_b, int64_t len_b,
                     int conts, const int64_t* cont_a, const int64_t* cont_b, int perm_len,
                     const int64_t* perm, int inc_c_len, const int64_t* inc_c, float* c,
                     int64_t offset_c, int64_t len_c, int n_dev, const int32_t* devices,
                     int32_t* err_codes, int64_t* err_info, int max_errs) {
  if (n_dev < 1) {
    t_last_error = "n_dev < 1";
    return GETT_E_INVALID_ARG;
  }
  return gett_impl<float>(true, rank_a, ext_a, inc_a, a, offset_a, len_a, rank_b, ext_b, inc_b, b,
                          offset_b, len_b, conts, cont_a, cont_b, perm_len, perm, inc_c_len, inc_c,
                          c, offset_c, len_c, nullptr, err_codes, err_info, max_errs, n_dev, devices);
}

int gett_set_devices(int n_dev, const int32_t* devices) {
  std::vector<int> v;
  if (n_dev < 0 || (n_dev > 0 && !devices)) return GETT_E_INVALID_ARG;
  if (n_dev > 0) {
    for (int i = 0; i < n_dev; ++i) {
      if (devices[i] < 0 || devices[i] >= kMaxDevices) return GETT_E_INVALID_ARG;
      v.push_back(devices[i]);
    }
  }
  std::lock_guard<std::mutex> lk(g_plan_mu);
  g_devices.swap(v);
  return 0;
}

int gett_set_multi(int strategy) {
  if (strategy < 0 || (strategy & 3) == 3 || strategy > 7) return GETT_E_INVALID_ARG;
  g_multi_force = strategy & 3;
  g_multi_stage = (strategy & 4) != 0;
  return 0;
}

const char* gett_last_multi(void) { return t_last_multi; }

int gett_multi_schedule(int rank_a, const int64_t* ext_a, const int64_t* inc_a, int64_t offset_a,
                        int64_t len_a, int rank_b, const int64_t* ext_b, const int64_t* inc_b,
                        int64_t offset_b, int64_t len_b, int conts, const int64_t* cont_a,
                        const int64_t* cont_b, int perm_len, const int64_t* perm, int inc_c_len,
                        const int64_t* inc_c, int64_t offset_c, int64_t len_c, int n_dev,
                        int strategy, int64_t* sched, int32_t* err_codes, int64_t* err_info,
                        int max_errs) {
  if (rank_a < 0 || rank_b < 0 || conts < 0 || perm_len < 0 || inc_c_len < 0 || n_dev < 1 || !sched ||
      strategy < 0 || strategy > 2) {
    t_last_error = "bad gett_multi_schedule arguments";
    return GETT_E_INVALID_ARG;
  }
  read_env();
  View va{rank_a, ext_a, inc_a, offset_a, len_a};
  View vb{rank_b, ext_b, inc_b, offset_b, len_b};
  Spec sp{conts, cont_a, cont_b, perm_len, perm, inc_c_len, inc_c};
  View vc{0, nullptr, nullptr, offset_c, len_c};
  std::vector<Error> errs = validate(va, vb, sp, CMode::Derived, vc);
  if (!errs.empty()) return fill_errors(errs, err_codes, err_info, max_errs);
  for (int i = 0; i < 4 + 2 * n_dev; ++i) sched[i] = 0;
  sched[1] = 1;
  sched[2] = sched[3] = -1;
  for (int d = 0; d < rank_a; ++d)
    if (ext_a[d] == 0) return 0;
  for (int d = 0; d < rank_b; ++d)
    if (ext_b[d] == 0) return 0;
  const Plan p = build_plan(va, vb, sp, offset_c, len_c);
  const MultiSched m = multi_schedule(p, va, vb, sp, n_dev, strategy);
  sched[0] = m.strategy;
  sched[1] = m.n;
  if (m.strategy == 1) {
    sched[2] = m.cut.owner;
    sched[3] = m.cut.dim;
  } else if (m.strategy == 2) {
    sched[3] = m.pair;
  }
  for (size_t i = 0; i < m.lo.size(); ++i) {
    sched[4 + 2 * i] = m.lo[i];
    sched[5 + 2 * i] = m.hi[i];
  }
  return 0;
}

#define GETT_COMPLEX_ENTRY(NAME, R, HOST, STREAM_PARAM, STREAM_ARG)                              \
  int NAME(int rank_a, const int64_t* ext_a, const int64_t* inc_a, const R* a, int64_t offset_a,   \
           int64_t len_a, int rank_b, const int64_t* ext_b, const int64_t* inc_b, const R* b,      \
           int64_t offset_b, int64_t len_b, int conts, const int64_t* cont_a,                      \
           const int64_t* cont_b, int perm_len, const int64_t* perm, int inc_c_len,                \
           const int64_t* inc_c, R* c, int64_t offset_c, int64_t len_c STREAM_PARAM,              \
           int32_t* err_codes, int64_t* err_info, int max_errs) {                                  \
    return gett_impl_complex<R>(HOST, rank_a, ext_a, inc_a, a, offset_a, len_a, rank_b, ext_b,     \
                                inc_b, b, offset_b, len_b, conts, cont_a, cont_b, perm_len, perm, \
                                inc_c_len, inc_c, c, offset_c, len_c, STREAM_ARG, err_codes,      \
                                err_info, max_errs);                                              \
  }
#define GETT_NO_STREAM_PARAM
#define GETT_STREAM_PARAM , void* stream
GETT_COMPLEX_ENTRY(gett_zgett, double, true, GETT_NO_STREAM_PARAM, nullptr)
GETT_COMPLEX_ENTRY(gett_cgett, float, true, GETT_NO_STREAM_PARAM, nullptr)
GETT_COMPLEX_ENTRY(gett_zgett_device, double, false, GETT_STREAM_PARAM, (cudaStream_t)stream)
GETT_COMPLEX_ENTRY(gett_cgett_device, float, false, GETT_STREAM_PARAM, (cudaStream_t)stream)

int gett_validate(int rank_a, const int64_t* ext_a, const int64_t* inc_a, int64_t offset_a,
                  int64_t len_a, int rank_b, const int64_t* ext_b, const int64_t* inc_b,
                  int64_t offset_b, int64_t len_b, int conts, const int64_t* cont_a,
                  const int64_t* cont_b, int perm_len, const int64_t* perm, int inc_c_len,
                  const int64_t* inc_c, int c_mode, int rank_cv, const int64_t* ext_cv,
                  const int64_t* inc_cv, int64_t offset_c, int64_t len_c, int32_t* err_codes,
                  int64_t* err_info, int max_errs) {
  if (rank_a < 0 || rank_b < 0 || conts < 0 || perm_len < 0 || inc_c_len < 0 || c_mode < 0 ||
      c_mode > 2 || (c_mode == 2 && rank_cv < 0)) {
    t_last_error = "bad validate arguments";
    return GETT_E_INVALID_ARG;
  }
  View va{rank_a, ext_a, inc_a, offset_a, len_a};
  View vb{rank_b, ext_b, inc_b, offset_b, len_b};
  Spec sp{conts, cont_a, cont_b, perm_len, perm, inc_c_len, inc_c};
  View vc{c_mode == 2 ? rank_cv : 0, ext_cv, inc_cv, offset_c, len_c};
  std::vector<Error> errs = validate(va, vb, sp, (CMode)c_mode, vc);
  return fill_errors(errs, err_codes, err_info, max_errs);
}

int gett_derive_output_extents(int rank_a, const int64_t* ext_a, int rank_b, const int64_t* ext_b,
                               int conts, const int64_t* cont_a, const int64_t* cont_b,
                               const int64_t* perm, int64_t* ext_c_out) {
  int rank_c = rank_a + rank_b - 2 * conts;
  if (rank_c < 0) return GETT_E_INVALID_ARG;
  int i = 0;
  auto contracted = [](const int64_t* idx, int n, int d) {
    for (int k = 0; k < n; ++k)
      if (idx[k] == d) return true;
    return false;
  };
  for (int d = 0; d < rank_a; ++d)
    if (!contracted(cont_a, conts, d)) {
      if (perm[i] < 0 || perm[i] >= rank_c) return GETT_E_INVALID_ARG;
      ext_c_out[perm[i++]] = ext_a[d];
    }
  for (int d = 0; d < rank_b; ++d)
    if (!contracted(cont_b, conts, d)) {
      if (perm[i] < 0 || perm[i] >= rank_c) return GETT_E_INVALID_ARG;
      ext_c_out[perm[i++]] = ext_b[d];
    }
  return rank_c;
}

int gett_zero_view_d(int rank, const int64_t* ext, const int64_t* inc, int64_t offset, int64_t len,
                     double* buf) {
  return zero_impl<double>(true, rank, ext, inc, offset, len, buf, nullptr);
}
int gett_zero_view_s(int rank, const int64_t* ext, const int64_t* inc, int64_t offset, int64_t len,
                     float* buf) {
  return zero_impl<float>(true, rank, ext, inc, offset, len, buf, nullptr);
}
int gett_zero_view_d_device(int rank, const int64_t* ext, const int64_t* inc, int64_t offset,
                            int64_t len, double* buf, void* stream) {
  return zero_impl<double>(false, rank, ext, inc, offset, len, buf, (cudaStream_t)stream);
}
int gett_zero_view_s_device(int rank, const int64_t* ext, const int64_t* inc, int64_t offset,
                            int64_t len, float* buf, void* stream) {
  return zero_impl<float>(false, rank, ext, inc, offset, len, buf, (cudaStream_t)stream);
}

int gett_pack(int rank, const int64_t* ext, const int64_t* inc, int64_t offset, int64_t len,
              int elem_bytes, const void* src, void* dst) {
  return pack_impl(true, rank, ext, inc, offset, len, elem_bytes, src, dst, nullptr);
}
int gett_pack_device(int rank, const int64_t* ext, const int64_t* inc, int64_t offset, int64_t len,
                     int elem_bytes, const void* src, void* dst, void* stream) {
  return pack_impl(false, rank, ext, inc, offset, len, elem_bytes, src, dst, (cudaStream_t)stream);
}

int gett_plan_create(char dtype, int rank_a, const int64_t* ext_a, const int64_t* inc_a, int64_t offset_a,
                     int64_t len_a, int rank_b, const int64_t* ext_b, const int64_t* inc_b,
                     int64_t offset_b, int64_t len_b, int conts, const int64_t* cont_a,
                     const int64_t* cont_b, int perm_len, const int64_t* perm, int inc_c_len,
                     const int64_t* inc_c, int64_t offset_c, int64_t len_c, int n_dev,
                     const int32_t* devices, gett_plan_t* out, int32_t* err_codes, int64_t* err_info,
                     int max_errs) {
  if (!out || (dtype != 'd' && dtype != 's') || rank_a < 0 || rank_b < 0 || conts < 0 || perm_len < 0 ||
      inc_c_len < 0 || offset_a < 0 || offset_b < 0 || offset_c < 0 || len_a < 0 || len_b < 0 ||
      len_c < 0 || n_dev < 0) {
    t_last_error = "bad gett_plan_create arguments (dtype 'd' or 's')";
    return GETT_E_INVALID_ARG;
  }
  *out = nullptr;
  read_env();
  std::vector<int> devs;
  int rc = check_devices(n_dev, devices, &devs);
  if (rc) return rc;
  View va{rank_a, ext_a, inc_a, offset_a, len_a};
  View vb{rank_b, ext_b, inc_b, offset_b, len_b};
  Spec sp{conts, cont_a, cont_b, perm_len, perm, inc_c_len, inc_c};
  View vc{0, nullptr, nullptr, offset_c, len_c};
  std::vector<Error> errs = validate(va, vb, sp, CMode::Derived, vc);
  if (!errs.empty()) return fill_errors(errs, err_codes, err_info, max_errs);
  std::unique_ptr<gett_plan_s> h(new gett_plan_s());
  h->dtype = dtype;
  h->ext_a.assign(ext_a, ext_a + rank_a);
  h->inc_a.assign(inc_a, inc_a + rank_a);
  h->ext_b.assign(ext_b, ext_b + rank_b);
  h->inc_b.assign(inc_b, inc_b + rank_b);
  h->cont_a.assign(cont_a, cont_a + conts);
  h->cont_b.assign(cont_b, cont_b + conts);
  h->perm.assign(perm, perm + perm_len);
  h->inc_c.assign(inc_c, inc_c + inc_c_len);
  h->off_a = offset_a;
  h->off_b = offset_b;
  h->off_c = offset_c;
  h->len_a = len_a;
  h->len_b = len_b;
  h->len_c = len_c;
  h->devs = devs;
  for (int d = 0; d < rank_a; ++d) h->empty = h->empty || ext_a[d] == 0;
  for (int d = 0; d < rank_b; ++d) h->empty = h->empty || ext_b[d] == 0;
  if (!h->empty) {
    DeviceGuard guard;
    if (!devs.empty()) CK(cudaSetDevice(devs[0]));
    CK(cudaGetDevice(&h->device));
    if ((rc = get_plan(dtype, h->va(), h->vb(), h->sp(), offset_c, len_c, &h->dp))) return rc;
  }
  *out = h.release();
  return 0;
}

int gett_execute(gett_plan_t plan, const void* a, const void* b, void* c) {
  if (!plan) return GETT_E_INVALID_ARG;
  return plan->dtype == 'd' ? execute_handle<double>(plan, true, a, b, c, nullptr)
                            : execute_handle<float>(plan, true, a, b, c, nullptr);
}

int gett_execute_device(gett_plan_t plan, const void* a, const void* b, void* c, void* stream) {
  if (!plan) return GETT_E_INVALID_ARG;
  return plan->dtype == 'd' ? execute_handle<double>(plan, false, a, b, c, (cudaStream_t)stream)
                            : execute_handle<float>(plan, false, a, b, c, (cudaStream_t)stream);
}

void gett_plan_destroy(gett_plan_t plan) { delete plan; }

int gett_set_kernel(const char* name) {
  if (!name) return GETT_E_INVALID_ARG;
  if (!strcmp(name, "auto")) g_mode = Mode::Auto;
  else if (!strcmp(name, "ref")) g_mode = Mode::Ref;
  else if (!strcmp(name, "tiled")) g_mode = Mode::Tiled;
  else if (!strcmp(name, "serial")) g_mode = Mode::Serial;
  else if (!strcmp(name, "ffma")) g_mode = Mode::Ffma;  // SGETT: register-tiled FFMA core
  else if (!strcmp(name, "dot")) g_mode = Mode::Dot;    // warp per output (few outputs, long K)
  else return GETT_E_INVALID_ARG;
  return 0;
}

int gett_set_split_k(int split) {
  if (split < 0) return GETT_E_INVALID_ARG;
  g_split = split;
  return 0;
}

int gett_set_pipeline(int slabs) {
  if (slabs < -1) return GETT_E_INVALID_ARG;
  g_pipeline_slabs = slabs;
  return 0;
}

int gett_set_stream_k(int on) {
  if (on != 0 && on != 1) return GETT_E_INVALID_ARG;
  g_stream_k = on != 0;
  return 0;
}

int gett_set_pair(int on) {
  if (on != 0 && on != 1) return GETT_E_INVALID_ARG;
  g_pair = on != 0;
  return 0;
}

int gett_set_complex_embed(int on) {
  if (on != 0 && on != 1) return GETT_E_INVALID_ARG;
  g_complex_4x = on == 0;
  return 0;
}

int gett_set_kr(int mode) {
  if (mode < 0 || (mode & 3) == 3 || mode > 31) return GETT_E_INVALID_ARG;
  g_kr = mode & 3;
  g_kr_fused = (mode & 4) != 0;
  g_kr_pair = (mode & 8) == 0;
  g_kr_mix = (mode & 16) == 0;
  return 0;
}

int gett_set_tma(int on) {
  if (on != 0 && on != 1) return GETT_E_INVALID_ARG;
  g_tma = on != 0;
  return 0;
}

int gett_set_wide(int mode) {
  if (mode < 0 || (mode & 3) == 3 || mode > 15) return GETT_E_INVALID_ARG;
  g_wide = mode & 3;
  g_wide_mix = (mode & 4) != 0;
  g_wide_tail = (mode & 8) == 0;
  return 0;
}

int gett_set_pdl(int on) {
  if (on != 0 && on != 1) return GETT_E_INVALID_ARG;
  g_launch_pdl = on;
  return 0;
}

int gett_set_bulk(int on) {
  if (on != 0 && on != 1) return GETT_E_INVALID_ARG;
  g_dgett_bulk = on != 0;
  return 0;
}

const char* gett_last_kernel(void) { return t_last_kernel; }
const char* gett_last_error(void) { return t_last_error.c_str(); }
int64_t gett_launch_count(void) { return g_launches; }

void gett_release_caches(void) {
  {
    std::lock_guard<std::mutex> lock(g_plan_mu);
    g_plans.map.clear();
    g_plans.lru.clear();
    g_last.dp.reset();
    g_last.key.clear();
  }
  int cur = -1;
  cudaGetDevice(&cur);
  for (int d = 0; d < kMaxDevices; ++d) {
    DevState& ds = g_dev[d];
    std::lock_guard<std::mutex> lk(ds.mu);
    if (ds.lanes.empty() && ds.sws.empty()) continue;
    cudaSetDevice(d);
    cudaDeviceSynchronize();  // kernels may still use the workspaces
    for (auto& L : ds.lanes)
      for (Scratch* s : {&L->a, &L->b, &L->c, &L->red})
        if (s->p) {
          cudaFree(s->p);
          s->p = nullptr;
          s->bytes = 0;
        }
    for (auto& sv : ds.sws)
      for (Scratch* s : {&sv.second.ws, &sv.second.part, &sv.second.flags, &sv.second.cx, &sv.second.krsync})
        if (s->p) cudaFree(s->p);
    ds.sws.clear();
  }
  if (cur >= 0) cudaSetDevice(cur);
}

// 1.02: gett_set_tma, gett_set_pair; 1.03: gett_set_complex_embed;
// 1.04: gett_{d,s}gett_multi, gett_set_devices, gett_set_multi, gett_last_multi,
//       gett_multi_schedule, gett_pack[_device], gett_set_kr,
// 1.05: gett_plan_create / gett_execute[_device] / gett_plan_destroy; 1.06: gett_set_bulk, gett_set_wide
// 1.07: gett_set_pdl; gett_set_kr + 16 (three tf32 MMAs instead of the mixed tf32 + bf16 split)
int gett_abi_version(void) { return 107; }

}  // extern "C"
