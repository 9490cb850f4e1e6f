// Rail calibration; pins in include/nezha/calibration.hpp.
// Restated independently in oracle/planner.py (calibrate).
#include "nezha/calibration.hpp"

#include <algorithm>
#include <cmath>
#include <stdexcept>

namespace nezha {

CalibratedProfile calibrate(int rail_id, ProtocolKind protocol, std::vector<std::pair<Bytes, Micros>> samples) {
  if (samples.size() < 2) throw std::invalid_argument("calibrate: needs at least 2 samples");
  std::sort(samples.begin(), samples.end());
  for (size_t i = 0; i < samples.size(); ++i) {
    if (!(samples[i].second > 0)) throw std::invalid_argument("calibrate: latencies must be positive");
    if (i && samples[i].first == samples[i - 1].first) throw std::invalid_argument("calibrate: repeated size");
  }
  // Weighted normal equations, w = 1 / y^2, summed in sample order.
  double sw = 0, sx = 0, sxx = 0, sy = 0, sxy = 0;
  for (const auto& [size, y] : samples) {
    const double x = static_cast<double>(size);
    const double w = 1.0 / (y * y);
    sw += w;
    sx += w * x;
    sxx += w * x * x;
    sy += w * y;
    sxy += w * x * y;
  }
  const double det = sw * sxx - sx * sx;
  CalibratedProfile out;
  out.profile.rail_id = rail_id;
  out.profile.protocol = protocol;
  double t = -1, c = -1;
  if (det > 0) {
    t = (sxx * sy - sx * sxy) / det;
    c = (sw * sxy - sx * sy) / det;
  }
  out.fit_t_setup_us = t;
  out.fit_us_per_byte = c;
  double worst = 0;
  for (const auto& [size, y] : samples) {
    worst = std::max(worst, std::fabs(t + c * static_cast<double>(size) - y) / y);
  }
  if (t >= 0 && c > 0 && worst <= 0.10) {
    out.profile.t_setup_us = t;
    out.profile.bandwidth_bps = 1e6 / c;
    out.max_rel_residual = worst;
  } else {
    out.interpolated = true;
    out.profile.efficiency_points = samples;
    out.profile.t_setup_us = samples.front().second;
    const double dx = static_cast<double>(samples.back().first - samples.front().first);
    const double dy = samples.back().second - samples.front().second;
    out.profile.bandwidth_bps = dy > 0 ? dx / (dy * 1e-6) : 1.0;
  }
  out.profile.validate();
  return out;
}

}  // namespace nezha
