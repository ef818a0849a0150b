// common.cuh — shared infrastructure of librpd_b200.so (sm_100a only).
//
// Conventions
//  * Every translation unit is compiled with --fmad=false: no a*b+c
//    contraction anywhere, so double/float expressions round exactly like the
//    reference's x86-64 SSE2 build (SURVEY.md §7 hard part 1).
//  * Errors inside the library are C++ exceptions (InvalidArg / Degenerate /
//    CudaFail) that the extern "C" layer (abi.cu) maps onto rpd_status.
//  * All device work of a context is ordered on ctx->stream.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "rpd_b200.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "librpd_b200 targets sm_100a only"
#endif

namespace rpdg {

struct InvalidArg : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct Degenerate : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CudaFail : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct Capacity : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define RPD_CK(x)                                                                    \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess)                                                           \
      throw ::rpdg::CudaFail(std::string(#x) + ": " + cudaGetErrorString(e_));       \
  } while (0)

// Debug / A-B switches (RPD_SKIP_STAGES, RPD_TMA_TYPES, ...) are read from the
// environment only in a build with -DRPD_DEBUG_KNOBS (`make DEBUG_KNOBS=1`).
// The product library ignores the environment entirely, so a caller's
// environment can never change its outputs.
inline const char* debug_knob(const char* name) {
#ifdef RPD_DEBUG_KNOBS
  return std::getenv(name);
#else
  (void)name;
  return nullptr;
#endif
}

// RPD_SYNC_DEBUG=1 in the environment (debug-knob builds) synchronises after every launch and
// names the failing call site (debugging only; never set in timed runs).
bool rpd_sync_debug();
#define RPD_LAUNCH_CHECK()                                                                 \
  do {                                                                                     \
    RPD_CK(cudaGetLastError());                                                            \
    if (::rpdg::rpd_sync_debug()) {                                                        \
      cudaError_t e2_ = cudaDeviceSynchronize();                                           \
      if (e2_ != cudaSuccess)                                                              \
        throw ::rpdg::CudaFail(std::string(__FILE__) + ":" + std::to_string(__LINE__) + \
                               ": " + cudaGetErrorString(e2_));                            \
    }                                                                                      \
  } while (0)

constexpr float kInvalid = -1.0f;  // types.hpp:21

inline int cdiv(long long a, long long b) { return int((a + b - 1) / b); }
__host__ __device__ inline int round_up(int a, int b) { return (a + b - 1) / b * b; }

// Device-side status word shared by the pipeline kernels: the first kernel
// that hits a reference exception condition records it; the host checks it
// once at the end of the call (no mid-pipeline synchronisation).
struct DevStatus {
  int code;    // 0 ok, else rpd_status
  int where;   // kind of failure, see status_message()
  long long aux;
};
enum StatusWhere : int {
  kWhereNone = 0,
  kWhereSampleBoot = 1,      // sample_observations n<3 in bootstrap fit
  kWhereFitBoot = 2,         // fit_line singular in bootstrap fit
  kWhereSamplePt = 3,
  kWhereFitPt = 4,
  kWhereThresholdEmpty = 5,  // find_road_threshold: all vectors excluded
  kWhereHistTooLarge = 6,
  kWhereSample = 7,          // standalone sample_observations
  kWhereFit = 8,             // standalone fit_line / estimate_roll / fit_road
};

__device__ inline void set_status(DevStatus* st, int code, int where, long long aux = 0) {
  if (atomicCAS(&st->code, 0, code) == 0) {
    st->where = where;
    st->aux = aux;
  }
}

// Road model as the device sees it: cos/sin travel with phi so every kernel
// evaluates road_disparity_at (types.hpp:39-41) with the same two values.
struct DevModel {
  double a0, a1, phi, c, s;
};

// road_disparity_at, types.hpp:39-41 — a0 + a1*(v*cos - u*sin), no FMA.
__host__ __device__ inline double road_at(const DevModel& m, double u, double v) {
  return m.a0 + m.a1 * (v * m.c - u * m.s);
}

// ----------------------------------------------------------- workspace ----
// Grow-only named device buffers.  Pointers stay stable until a request
// exceeds the current capacity, so captured CUDA graphs stay valid for a
// fixed problem shape.
class Workspace {
 public:
  ~Workspace() { release(); }
  void release() {
    for (auto& kv : bufs_)
      if (kv.second.p) cudaFree(kv.second.p);
    bufs_.clear();
  }
  template <typename T>
  T* get(const std::string& name, size_t count) {
    Buf& b = bufs_[name];
    const size_t bytes = std::max<size_t>(count * sizeof(T), 16);
    if (b.bytes < bytes) {
      if (b.p) RPD_CK(cudaFree(b.p));
      b.p = nullptr;
      b.bytes = 0;
#ifdef RPD_DEBUG_KNOBS
      // checked build: no headroom, a guard zone right after the requested
      // bytes that rpd_debug_guard_check verifies
      const size_t want = bytes;
      const size_t alloc = want + kGuardBytes;
#else
      const size_t want = bytes + bytes / 8;  // headroom for small shape drift
      const size_t alloc = want;
#endif
      if (cudaMalloc(&b.p, alloc) != cudaSuccess) {
        cudaGetLastError();
        throw CudaFail("device allocation of " + std::to_string(alloc) + " bytes failed (" +
                       name + ")");
      }
#ifdef RPD_DEBUG_KNOBS
      RPD_CK(cudaMemset(static_cast<char*>(b.p) + want, kGuardByte, kGuardBytes));
#endif
      b.bytes = want;
      ++generation_;
    }
    return static_cast<T*>(b.p);
  }
  unsigned generation() const { return generation_; }

  // Checked build: number of guard bytes overwritten (first offender in *who).
  long long check_guards(std::string* who) const {
#ifdef RPD_DEBUG_KNOBS
    long long bad = 0;
    std::vector<unsigned char> h(kGuardBytes);
    for (const auto& kv : bufs_) {
      if (!kv.second.p) continue;
      RPD_CK(cudaMemcpy(h.data(), static_cast<const char*>(kv.second.p) + kv.second.bytes,
                        kGuardBytes, cudaMemcpyDeviceToHost));
      long long n = 0;
      for (unsigned char c : h) n += c != kGuardByte;
      if (n && who && who->empty()) *who = kv.first;
      bad += n;
    }
    return bad;
#else
    (void)who;
    return -1;
#endif
  }

 private:
  static constexpr size_t kGuardBytes = 4096;
  static constexpr unsigned char kGuardByte = 0xA5;
  struct Buf {
    void* p = nullptr;
    size_t bytes = 0;
  };
  std::map<std::string, Buf> bufs_;
  unsigned generation_ = 0;
};

// Pinned host staging area (grow-only).
class PinnedHost {
 public:
  ~PinnedHost() {
    if (p_) cudaFreeHost(p_);
  }
  void* get(size_t bytes) {
    if (bytes > bytes_) {
      if (p_) RPD_CK(cudaFreeHost(p_));
      p_ = nullptr;
      RPD_CK(cudaMallocHost(&p_, bytes));
      bytes_ = bytes;
    }
    return p_;
  }

 private:
  void* p_ = nullptr;
  size_t bytes_ = 0;
};

}  // namespace rpdg

struct rpd_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  std::string err;
  rpdg::Workspace ws;
  rpdg::PinnedHost pinned;
  rpdg::DevStatus* status = nullptr;  // device
  cudaEvent_t ev[RPD_NUM_STAGES + 1] = {};
  int sm_count = 148;
  void* pipeline = nullptr;  // rpdg::PipelineState (pipeline.cu)
  // measurement (rpd_ctx_set_profiling / rpd_ctx_stats)
  bool profile = false;
  int agg_pass = 0;                       // aggregation launches recorded this frame
  cudaEvent_t agg_ev[2][2] = {};          // [pass][start/end]
  double agg_alg_bytes[2] = {0, 0};
  double agg_cells[2] = {0, 0};
  int kernels_last_frame = 0;
  int graph_replayed = 0;
  int last_agg_kernel = 0;  // rpdg::AggImpl of the last aggregation
  void* agg_flags_zeroed = nullptr;  // segmented aggregation: flag buffer known to be zero
  int agg_flags_words = 0;
  void* scan_zeroed = nullptr;          // scan descriptors known to be zero (scan.cu)
  long long scan_zeroed_tiles = 0;
  void* scan_ctl_zeroed = nullptr;
  int agg_segmented_ctas = 0;                  // last aggregation launch
  unsigned long long* agg_reruns = nullptr;    // device counter (workspace)
  unsigned long long* slic_tiles = nullptr;    // device counters {tiles assigned, skipped, centres moved, pixels changed}
};

namespace rpdg {

// Host-side helpers shared by the translation units ---------------------
void reset_status(rpd_ctx* ctx);
// Synchronises the stream and throws the recorded device status, if any.
void sync_and_check(rpd_ctx* ctx);
void check_status(const DevStatus& h);  // throws the status' exception
DevModel host_model(const rpd_road_model& m);  // cos/sin on the host (glibc)
void pipeline_forget(rpd_ctx* ctx);           // releases captured graphs
// Records `ev` on ctx->stream; inside a stream capture it becomes an external
// event-record node so the event is really recorded on every graph replay.
void record_event(rpd_ctx* ctx, cudaEvent_t ev);
// out[i] = in[0] + ... + in[i-1] on ctx->stream, one launch (scan.cu).
void scan_exclusive_i32(rpd_ctx* ctx, const int* in, int* out, long long n);

}  // namespace rpdg
