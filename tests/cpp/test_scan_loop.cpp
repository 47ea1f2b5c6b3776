// The reference's own stereo_scan loop shape (pipeline.hpp:157-190: OpenMP
// over rows, schedule(dynamic, 4), one search_depth per masked pixel, results
// slotted per pixel and compacted in raster order) compiled against the
// drop-in headers, so every search_depth call runs on the GPU; then the same
// frame through the one-launch drop-in dfuse::stereo_scan, and
// update_semidense. Reports per frame the observation count, the image
// uploads the frame cost (dfuse_image_uploads) and whether the two scans
// agree bit for bit; finally the semi-dense map. Driven by
// tests/test_cpp_dropin.py, which checks the map against the oracle.
//
// usage: test_scan_loop <input.bin> <output.bin>
#include <omp.h>

#include <cstdio>
#include <cstring>
#include <fstream>
#include <vector>

#include "dfuse/stereo_scan.hpp"

using namespace dfuse;

template <class T>
static void rd(std::ifstream& f, T* p, size_t n) {
  f.read(reinterpret_cast<char*>(p), sizeof(T) * n);
  if (!f) throw std::runtime_error("short input");
}
template <class T>
static void wr(std::ofstream& f, const T* p, size_t n) {
  f.write(reinterpret_cast<const char*>(p), sizeof(T) * n);
}

int main(int argc, char** argv) {
  if (argc != 3) return 2;
  std::ifstream in(argv[1], std::ios::binary);
  int32_t hdr[3];
  rd(in, hdr, 3);
  const int W = hdr[0], H = hdr[1], nframes = hdr[2];
  double k[4], sc[3];
  rd(in, k, 4);
  rd(in, sc, 3);
  const CameraIntrinsics K{k[0], k[1], k[2], k[3], W, H};
  const SearchConfig cfg{sc[0], sc[1], sc[2]};
  const size_t P = static_cast<size_t>(W) * H;
  IntensityImage I0(W, H);
  rd(in, I0.raster().data(), P);
  const Pose T0 = Pose::identity();
  const Mask texture = texture_mask(I0, 0.02);
  SemiDenseMap map = SemiDenseMap::empty(W, H);
  std::ofstream out(argv[2], std::ios::binary);
  for (int f = 0; f < nframes; ++f) {
    double q[4], t[3];
    rd(in, q, 4);
    rd(in, t, 3);
    Pose T1;
    T1.rotation = Eigen::Quaterniond(q[0], q[1], q[2], q[3]);
    T1.translation = Eigen::Vector3d(t[0], t[1], t[2]);
    IntensityImage I1(W, H);
    rd(in, I1.raster().data(), P);
    int64_t up0 = 0, up1 = 0;
    dfuse_image_uploads(&up0, nullptr);
    // ---- pipeline.hpp:159-189, verbatim in shape
    const EpipolarGeometry g = make_epipolar_geometry(T0, T1, K);
    std::vector<EpipolarObservation> obs;
    if (!(g.t_10.norm() < 1e-12)) {
      std::vector<EpipolarObservation> slots(P);
      std::vector<std::uint8_t> got(P, 0);
#pragma omp parallel for schedule(dynamic, 4)
      for (int y = 0; y < H; ++y) {
        for (int x = 0; x < W; ++x) {
          if (!texture.at(x, y)) continue;
          const std::size_t i = texture.index(x, y);
          std::optional<DepthPrior> prior;
          if (map.valid[i]) prior = DepthPrior{map.depth[i], std::sqrt(map.variance[i])};
          const EpipolarResult r =
              search_depth(g, I0, I1, PixelCoord{static_cast<double>(x), static_cast<double>(y)},
                           prior, cfg);
          if (r.ok()) {
            slots[i] = r.obs;
            got[i] = 1;
          }
        }
      }
      obs.reserve(P / 4);
      for (std::size_t i = 0; i < P; ++i)
        if (got[i]) obs.push_back(slots[i]);
    }
    // ---- the one-launch drop-in on the same inputs
    const std::vector<EpipolarObservation> obs2 = stereo_scan(g, I0, I1, texture, map, cfg);
    dfuse_image_uploads(&up1, nullptr);
    const int32_t same = obs.size() == obs2.size() &&
                         (obs.empty() || std::memcmp(obs.data(), obs2.data(),
                                                     obs.size() * sizeof(EpipolarObservation)) == 0);
    if (!obs.empty()) map = update_semidense(std::move(map), obs);  // pipeline.hpp:209-212
    const int32_t rec[4] = {static_cast<int32_t>(obs.size()), static_cast<int32_t>(up1 - up0), same,
                            omp_get_max_threads()};
    wr(out, rec, 4);
    std::printf("frame %d: %zu observations, %lld image uploads, one-launch scan %s\n", f,
                obs.size(), static_cast<long long>(up1 - up0), same ? "identical" : "DIFFERENT");
  }
  wr(out, map.depth.data(), P);
  wr(out, map.variance.data(), P);
  wr(out, map.valid.data(), P);
  const int32_t cnt = map.inlier_count;
  wr(out, &cnt, 1);
  return 0;
}
