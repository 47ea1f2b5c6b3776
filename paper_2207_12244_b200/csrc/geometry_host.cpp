// geometry_host.cpp -- per-frame-pair geometry on the host:
// make_epipolar_geometry (semidense.hpp:101-106) over Pose/compose
// (geometry.hpp:44-67). 15 doubles per frame pair, so it stays on the CPU;
// it uses the same quaternion code (include/compat/Eigen) the oracle build of
// the reference uses, which makes the geometry bit-identical on both paths.
#include <Eigen/Core>
#include <Eigen/Geometry>

#include "../../include/dfuse_cuda.h"

namespace {

struct Pose {
  Eigen::Quaterniond rotation;
  Eigen::Vector3d translation;
  Pose inverse() const {  // geometry.hpp:52-55
    const Eigen::Quaterniond qi = rotation.conjugate();
    return {qi, -(qi * translation)};
  }
};

Pose compose(const Pose& a, const Pose& b) {  // geometry.hpp:65-67
  return {(a.rotation * b.rotation).normalized(), a.rotation * b.translation + a.translation};
}

}  // namespace

extern "C" int dfuse_make_epipolar_geometry(const double q0[4], const double t0[3],
                                            const double q1[4], const double t1[3],
                                            const dfuse_intrinsics* K, dfuse_epigeom* out) {
  if (!q0 || !t0 || !q1 || !t1 || !K || !out) return DFUSE_E_INVALID_ARGUMENT;
  const Pose T0{Eigen::Quaterniond(q0[0], q0[1], q0[2], q0[3]),
                Eigen::Vector3d(t0[0], t0[1], t0[2])};
  const Pose T1{Eigen::Quaterniond(q1[0], q1[1], q1[2], q1[3]),
                Eigen::Vector3d(t1[0], t1[1], t1[2])};
  const Pose T10 = compose(T1.inverse(), T0);
  const Pose T01 = compose(T0.inverse(), T1);
  const Eigen::Matrix3d R = T10.rotation.toRotationMatrix();
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) out->R_10[3 * r + c] = R(r, c);
  for (int i = 0; i < 3; ++i) {
    out->t_10[i] = T10.translation(i);
    out->t_01[i] = T01.translation(i);
  }
  out->K = *K;
  return DFUSE_OK;
}
