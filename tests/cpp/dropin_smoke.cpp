// C++ drop-in smoke test: a handful of the reference's own unit-test known
// answers (test_sgm.cpp, test_perspective.cpp, test_segmentation.cpp) written
// against rpd_b200.hpp exactly as they are written against rpd::.  Compiled
// on CPU by tests/test_abi.py; run on the GPU by tests/test_cpp_dropin.py.
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "rpd_b200.hpp"

using namespace rpd_b200;

static int failures = 0;
#define CHECK(x)                                                       \
  do {                                                                 \
    if (!(x)) {                                                        \
      std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #x);         \
      ++failures;                                                      \
    }                                                                  \
  } while (0)

int main() {
  {  // test_sgm.cpp:86-93
    GrayImage img = GrayImage::Constant(8, 8, 100.0f);
    CostVolume vol = census_cost_volume(img, img, 3, 5);
    for (int v = 0; v < 8; ++v)
      for (int u = 3; u < 8; ++u)
        for (int d = 0; d <= 3; ++d) CHECK(vol.at(v, u, d) == 0.0f);
    CHECK(vol.at(0, 0, 1) == 24.0f);
  }
  {  // test_sgm.cpp:158-181 parabola
    CostVolume vol(1, 1, 6);
    const float c[7] = {40, 30, 4, 2, 4, 31, 41};
    for (int d = 0; d <= 6; ++d) vol.at(0, 0, d) = c[d];
    CHECK(std::fabs(select_disparity(vol)(0, 0) - 3.0f) < 1e-6f);
  }
  {  // test_perspective.cpp:36-61
    GrayImage img(1, 4);
    img(0, 0) = 10; img(0, 1) = 20; img(0, 2) = 30; img(0, 3) = 40;
    WarpResult w1 = warp_right_image(img, {{1.0}, 0.0});
    CHECK(w1.image(0, 0) == 0.0f && w1.in_view(0, 0) == 0 && w1.image(0, 1) == 10.0f);
  }
  {  // test_segmentation.cpp:294-299 diagonal touch
    LabelMap m = LabelMap::Zero(3, 3);
    m(0, 0) = 1;
    m(1, 1) = 1;
    LabelMap a = connected_components(m, 8), b = connected_components(m, 4);
    int ma = 0, mb = 0;
    for (int x : a.data) ma = std::max(ma, x);
    for (int x : b.data) mb = std::max(mb, x);
    CHECK(ma == 1 && mb == 2);
  }
  {  // test_sgm.cpp:224-230 error behaviour
    GrayImage a = GrayImage::Zero(4, 8), b = GrayImage::Zero(4, 9);
    bool threw = false;
    try {
      census_cost_volume(a, b, 2, 5);
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    CHECK(threw);
  }
  {  // full pipeline on a textured pair: left(u) = right(u - 6)
    const int h = 96, w = 160;
    GrayImage left(h, w), right(h, w);
    unsigned s = 12345;
    for (int v = 0; v < h; ++v)
      for (int u = 0; u < w; ++u) {
        s = s * 1103515245u + 12345u;
        right(v, u) = float((s >> 16) & 255);
      }
    for (int v = 0; v < h; ++v)
      for (int u = 0; u < w; ++u) left(v, u) = right(v, std::max(0, u - 6));
    PipelineConfig cfg;
    cfg.d_max = 31;
    cfg.superpixels = 100;
    try {
      DetectResult r = detect_potholes_pipeline(left, right, cfg);
      CHECK(r.superpixels.count > 50 && r.stage_times.size() == 7);
    } catch (const DegenerateFitError& e) {
      std::printf("degenerate fit (acceptable for a planar-free pair): %s\n", e.what());
    }
  }
  {  // test_evaluation.cpp:10-35 / :97-108 (pep, rmse, pixel metrics)
    DisparityMap gt = DisparityMap::Constant(2, 5, 10.0f);
    DisparityMap est = gt;
    est(0, 0) = 13.5f;
    est(0, 1) = 12.0f;
    est(1, 0) = kInvalidDisparity;
    gt(1, 1) = kInvalidDisparity;
    CHECK(std::fabs(pep(est, gt, 2.0) - 100.0 / 8.0) < 1e-12);
    DisparityMap g1 = DisparityMap::Constant(1, 4, 5.0f);
    DisparityMap e1(1, 4);
    e1(0, 0) = 5.0f; e1(0, 1) = 8.0f; e1(0, 2) = 1.0f; e1(0, 3) = kInvalidDisparity;
    CHECK(std::fabs(rmse(e1, g1) - std::sqrt(25.0 / 3.0)) < 1e-12);
    LabelMap pred(2, 4), gtm(2, 4);
    const int pv[8] = {1, 1, 0, 0, 2, 0, 0, 0}, gv[8] = {1, 0, 1, 0, 1, 1, 0, 0};
    for (int i = 0; i < 8; ++i) { pred(i / 4, i % 4) = pv[i]; gtm(i / 4, i % 4) = gv[i]; }
    const PixelMetrics m = pixel_metrics(pred, gtm);
    CHECK(m.counts.n_tp == 2 && m.counts.n_fp == 1 && m.counts.n_fn == 2 && m.counts.n_tn == 3);
    CHECK(instance_metrics(pred, pred).correct == 2);
  }
  {  // test_road_geometry.cpp:209-225 (reproject)
    StereoRig rig{700.0, 0.12, 320.0, 240.0};
    DisparityMap d = DisparityMap::Constant(2, 2, kInvalidDisparity);
    d(0, 0) = 7.0f;
    PointCloud c = reproject(d, rig);
    CHECK(c.size() == 1 && std::fabs(c[0].z - 12.0f) < 1e-5f);
    CHECK(closest_distance_error(c, c) == 0.0);
  }
  {  // test_synth.cpp:46-61, 131-147
    SceneSpec spec;
    spec.width = 160;
    spec.height = 120;
    spec.texture_seed = 42;
    spec.potholes.push_back({80.0, 60.0, 18.0, 12.0, 3.0});
    SceneTruth sc = generate_scene(spec);
    CHECK(sc.gt_mask(60, 80) == 1 && sc.gt_mask(60, 100) == 0);
    CHECK(std::fabs(sc.gt_disparity(60, 80) - (road_disparity_at({5.0, 0.08, 0.0}, 80, 60) - 3.0)) <
          1e-5);
    std::vector<SceneTruth> batch = scene_batch(2, 900);
    CHECK(batch.size() == 2 && !batch[0].spec.potholes.empty());
    CHECK(batch[1].left.rows() == 480 && batch[1].left.cols() == 640);
  }
  std::printf("%s (%d failures)\n", failures ? "FAILED" : "OK", failures);
  return failures ? 1 : 0;
}
