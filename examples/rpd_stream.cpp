// rpd_stream.cpp — a native C++ frame server on the C-ABI (no Python, no
// torch): K pipeline contexts (one CUDA stream, workspace and captured graph
// each) kept busy by T host threads through the streaming entry points
// (rpd_detect_async_host_u8: async H2D from pinned memory + the frame;
// rpd_detect_fetch: D2H of the outputs into pinned buffers).  Frames are
// scene_batch scenes (synth.cpp:151-192) generated with the library itself.
//
//   g++ -std=c++17 -O2 -I include examples/rpd_stream.cpp -o rpd_stream
//       -L paper_2012_10802_b200/_lib -lrpd_b200 -Wl,-rpath,<that dir> -lpthread
//   ./rpd_stream [frames] [contexts] [threads] [scenes]
// Prints one JSON line: frames/s, and each scene's pothole count (the same on
// every pass through the scene: the pipeline is deterministic).
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

#include "rpd_b200.h"

namespace {

void check(rpd_ctx* ctx, rpd_status st, const char* what) {
  if (st != RPD_OK) {
    std::fprintf(stderr, "%s failed: status %d (%s)\n", what, int(st), ctx ? rpd_last_error(ctx) : "");
    std::exit(1);
  }
}

struct Outputs {
  float* d1 = nullptr;
  float* d2 = nullptr;
  int32_t* labels = nullptr;
};

}  // namespace

int main(int argc, char** argv) {
  const int frames = argc > 1 ? std::atoi(argv[1]) : 256;
  const int nctx = argc > 2 ? std::atoi(argv[2]) : 16;
  const int nthr = argc > 3 ? std::atoi(argv[3]) : 4;
  const int nscenes = argc > 4 ? std::atoi(argv[4]) : 8;
  if (frames < 1 || nctx < 1 || nthr < 1 || nscenes < 1) {
    std::fprintf(stderr, "usage: rpd_stream [frames] [contexts] [threads] [scenes]\n");
    return 2;
  }

  std::vector<rpd_ctx*> ctx(static_cast<size_t>(nctx), nullptr);
  for (auto& c : ctx) check(nullptr, rpd_ctx_create(0, 0, 0, 0, &c), "rpd_ctx_create");

  // scenes of the acceptance batch (640 x 480), converted to the u8 pairs a
  // camera delivers, in pinned host memory
  rpd_batch_ranges ranges;
  rpd_batch_ranges_default(&ranges);
  rpd_scene_spec spec;
  rpd_pothole_spec holes[3];
  check(ctx[0], rpd_scene_batch_spec(7100u, 0, &ranges, &spec, holes), "rpd_scene_batch_spec");
  const int w = spec.width, h = spec.height;
  const size_t n = size_t(w) * size_t(h);
  std::vector<uint8_t*> left(static_cast<size_t>(nscenes), nullptr);
  std::vector<uint8_t*> right(static_cast<size_t>(nscenes), nullptr);
  {
    std::vector<float> fl(n), fr(n);
    for (int i = 0; i < nscenes; ++i) {
      check(ctx[0], rpd_scene_batch_spec(7100u, i, &ranges, &spec, holes), "rpd_scene_batch_spec");
      check(ctx[0], rpd_generate_scene(ctx[0], &spec, fl.data(), fr.data(), nullptr, nullptr),
            "rpd_generate_scene");
      void* pl = nullptr;
      void* pr = nullptr;
      check(nullptr, rpd_host_alloc(n, &pl), "rpd_host_alloc");
      check(nullptr, rpd_host_alloc(n, &pr), "rpd_host_alloc");
      left[size_t(i)] = static_cast<uint8_t*>(pl);
      right[size_t(i)] = static_cast<uint8_t*>(pr);
      for (size_t p = 0; p < n; ++p) {
        left[size_t(i)][p] = uint8_t(fl[p]);
        right[size_t(i)][p] = uint8_t(fr[p]);
      }
    }
  }

  rpd_config cfg;
  rpd_config_default(&cfg);
  cfg.delta_pd = 0.48;  // the acceptance gate's settings (acceptance.cpp:231)
  cfg.superpixels = 2400;
  check(ctx[0], rpd_config_validate(ctx[0], &cfg), "rpd_config_validate");

  // per-context pinned output buffers (what a server writes to disk / sends)
  std::vector<Outputs> outs(static_cast<size_t>(nctx));
  for (auto& o : outs) {
    void* p = nullptr;
    check(nullptr, rpd_host_alloc(n * sizeof(float), &p), "rpd_host_alloc");
    o.d1 = static_cast<float*>(p);
    check(nullptr, rpd_host_alloc(n * sizeof(float), &p), "rpd_host_alloc");
    o.d2 = static_cast<float*>(p);
    check(nullptr, rpd_host_alloc(n * sizeof(int32_t), &p), "rpd_host_alloc");
    o.labels = static_cast<int32_t*>(p);
  }
  std::vector<std::atomic<int>> potholes(static_cast<size_t>(nscenes));
  for (auto& x : potholes) x = -1;
  std::atomic<int> inconsistent{0};

  auto serve = [&](int count) {
    std::atomic<int> ticket{0};
    auto work = [&](int j) {
      std::vector<int> mine;
      for (int c = j; c < nctx; c += nthr) mine.push_back(c);
      std::vector<int> scene_of(static_cast<size_t>(nctx), -1), busy;
      auto enqueue = [&](int c) {
        const int q = ticket.fetch_add(1);
        if (q >= count) return false;
        const int s = q % nscenes;
        scene_of[size_t(c)] = s;
        check(ctx[size_t(c)],
              rpd_detect_async_host_u8(ctx[size_t(c)], left[size_t(s)], right[size_t(s)], h, w, &cfg),
              "rpd_detect_async_host_u8");
        return true;
      };
      for (int c : mine)
        if (enqueue(c)) busy.push_back(c);
      while (!busy.empty()) {
        const int c = busy.front();
        busy.erase(busy.begin());
        rpd_detect_out o;
        std::memset(&o, 0, sizeof(o));
        o.d1 = outs[size_t(c)].d1;
        o.d2 = outs[size_t(c)].d2;
        o.labels = outs[size_t(c)].labels;
        check(ctx[size_t(c)], rpd_detect_fetch(ctx[size_t(c)], &o), "rpd_detect_fetch");
        int expect = -1;
        if (!potholes[size_t(scene_of[size_t(c)])].compare_exchange_strong(expect, o.n_potholes) &&
            expect != o.n_potholes)
          ++inconsistent;
        if (enqueue(c)) busy.push_back(c);
      }
    };
    std::vector<std::thread> th;
    for (int j = 0; j < nthr; ++j) th.emplace_back(work, j);
    for (auto& t : th) t.join();
  };

  serve(nctx);  // warm-up: every context captures its frame graph
  const auto t0 = std::chrono::steady_clock::now();
  serve(frames);
  const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();

  std::printf("{\"frames\": %d, \"contexts\": %d, \"threads\": %d, \"width\": %d, \"height\": %d, "
              "\"frames_per_s\": %.1f, \"inconsistent\": %d, \"potholes\": [",
              frames, nctx, nthr, w, h, frames / s, inconsistent.load());
  for (int i = 0; i < nscenes; ++i) std::printf("%s%d", i ? ", " : "", potholes[size_t(i)].load());
  std::printf("]}\n");

  for (auto& o : outs) {
    rpd_host_free(o.d1);
    rpd_host_free(o.d2);
    rpd_host_free(o.labels);
  }
  for (int i = 0; i < nscenes; ++i) {
    rpd_host_free(left[size_t(i)]);
    rpd_host_free(right[size_t(i)]);
  }
  for (auto* c : ctx) rpd_ctx_destroy(c);
  return inconsistent.load() == 0 ? 0 : 1;
}
