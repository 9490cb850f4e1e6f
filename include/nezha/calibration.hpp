// nezha/calibration.hpp — rail calibration from single-rail latency samples
// (SPEC.md:434-446 `calibrate(samples) -> CalibratedProfile`, Table 1).
//
// The engine measures each rail alone over a size sweep at startup and feeds
// the samples here. Pinned (P15; the SPEC leaves the fit open):
//  - latency(S) = t_setup + c·S fitted by least squares on RELATIVE
//    residuals (weights 1/y_i^2), since the acceptance bound is relative;
//  - the fit is kept when t_setup >= 0, c > 0 and every sample is reproduced
//    within 10 %; the profile is then parametric
//    (bandwidth_bps = 1e6 / c);
//  - otherwise the samples become the profile's interpolation table (exact;
//    SPEC.md:443 fallback), t_setup = the smallest sample's latency and
//    bandwidth = the end-to-end slope, both for reporting only.
#pragma once

#include <utility>
#include <vector>

#include "nezha/core/types.hpp"

namespace nezha {

struct CalibratedProfile {
  RailProfile profile;
  bool interpolated = false;    // true: profile.efficiency_points carries the samples
  double max_rel_residual = 0;  // of the parametric fit (0 when interpolated)
  Micros fit_t_setup_us = 0;    // the least-squares solution, kept or not
  double fit_us_per_byte = 0;
};

/// std::invalid_argument on fewer than 2 samples, non-positive latency or
/// repeated sizes; an interpolation table that is not strictly increasing
/// fails RailProfile::validate.
CalibratedProfile calibrate(int rail_id, ProtocolKind protocol, std::vector<std::pair<Bytes, Micros>> samples);

}  // namespace nezha
