// Engine startup calibration (P13/P15): each rail's
// latency profile alone and with every rail busy, the fork/join sync
// overhead, and (tune_budgets) the measured CTA budgets and protocol
// crossovers of the SM-driven rails.
#include "engine_impl.h"

using nz::fail;

void nz_engine::tuneBudgets(uint64_t maxb, cudaEvent_t e0, cudaEvent_t e1) {
  if (comm->world == 1) return;
  const uint64_t s = std::min<uint64_t>(uint64_t{64} << 20, maxb) & ~uint64_t{4095};
  if (s <= (uint64_t{4} << 20)) return;  // must be past the one-shot (LL) ceiling
  for (size_t i = 0; i < rails.size(); ++i) {
    nz_rail* r = rails[i];
    if (specs[i].sm_budget > 0) continue;
    std::vector<int> cands;
    if (r->kind == NZ_RAIL_NVLS) cands = {16, 32, 64};
    if (r->kind == NZ_RAIL_SM) cands = {32, 64, 128};
    if (cands.empty()) continue;
    const uint64_t C = nezha::defaultChunkBytes(s, comm->world, algo);
    std::vector<double> t(cands.size());
    for (size_t k = 0; k < cands.size(); ++k) {
      r->sm_budget = std::min(cands[k], comm->sm_count);
      for (int w = 0; w < 2; ++w) nz::railAllreduce(r, ub_in, ub_out, 0, s, C, 0, UINT64_MAX, NZ_F32, 0, -1, r->stream);
      NZ_CUDA(cudaEventRecord(e0, r->stream));
      for (int it = 0; it < 5; ++it) nz::railAllreduce(r, ub_in, ub_out, 0, s, C, 0, UINT64_MAX, NZ_F32, 0, -1, r->stream);
      NZ_CUDA(cudaEventRecord(e1, r->stream));
      NZ_CUDA(cudaEventSynchronize(e1));
      float ms = 0;
      NZ_CUDA(cudaEventElapsedTime(&ms, e0, e1));
      t[k] = ms;
    }
    const auto msgs = nz::exchange(comm, t.data(), t.size() * sizeof(double), {});
    for (int rk = 0; rk < comm->world; ++rk) {
      const double* v = reinterpret_cast<const double*>(msgs[rk].data.data());
      for (size_t k = 0; k < t.size(); ++k) t[k] = std::max(t[k], v[k]);
    }
    size_t best = 0;
    for (size_t k = 1; k < t.size(); ++k)
      if (t[k] < t[best] * 0.97) best = k;
    r->sm_budget = std::min(cands[best], comm->sm_count);
  }
}

void nz_engine::tunePaths(uint64_t maxb, cudaEvent_t e0, cudaEvent_t e1) {
  if (comm->world == 1) return;
  for (size_t i = 0; i < rails.size(); ++i) {
    nz_rail* r = rails[i];
    if (r->ll_cap == 0) continue;
    std::vector<uint64_t> sizes;
    for (uint64_t sz = 64 << 10; sz <= std::min<uint64_t>(uint64_t{4} << 20, maxb); sz *= 2) sizes.push_back(sz);
    if (sizes.empty()) continue;
    // times[3k + v]: v = 0 LL, 2 two-shot (1, the staged one-shot of round 1,
    // is gone: never applicable); huge when not applicable.
    std::vector<double> t(sizes.size() * 3, 1e30);
    for (size_t k = 0; k < sizes.size(); ++k) {
      const uint64_t s = sizes[k];
      const uint64_t C = nezha::defaultChunkBytes(s, comm->world, algo);
      for (int v : {0, 2}) {
        if (v == 0 && s > r->ll_cap) continue;
        r->ll_max = v == 0 ? r->ll_cap : 0;
        for (int w = 0; w < 3; ++w) nz::railAllreduce(r, ub_in, ub_out, 0, s, C, 0, UINT64_MAX, NZ_F32, 0, -1, r->stream);
        NZ_CUDA(cudaEventRecord(e0, r->stream));
        for (int it = 0; it < 20; ++it) nz::railAllreduce(r, ub_in, ub_out, 0, s, C, 0, UINT64_MAX, NZ_F32, 0, -1, r->stream);
        NZ_CUDA(cudaEventRecord(e1, r->stream));
        NZ_CUDA(cudaEventSynchronize(e1));
        float ms = 0;
        NZ_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        t[k * 3 + v] = ms;
      }
    }
    const auto msgs = nz::exchange(comm, t.data(), t.size() * sizeof(double), {});
    for (int rk = 0; rk < comm->world; ++rk) {
      const double* v = reinterpret_cast<const double*>(msgs[rk].data.data());
      for (size_t j = 0; j < t.size(); ++j) t[j] = std::max(t[j], v[j]);
    }
    r->ll_max = nezha::choosePathCeilings(sizes, t, r->ll_cap, 0).first;
  }
}

void nz_engine::calibrate() {
  const uint64_t maxb = std::max<uint64_t>(cfg.calibrate_max_bytes, 1 << 16);
  ensureUnbound(maxb);
  const int world = comm->world;
  std::vector<uint64_t> sizes;
  for (uint64_t s = 4096; s <= maxb; s *= 4) sizes.push_back(s);
  cudaEvent_t e0 = event(), e1 = event();
  if (cfg.tune_budgets) {
    tuneBudgets(maxb, e0, e1);
    tunePaths(maxb, e0, e1);
  }
  std::vector<nezha::RailProfile> profiles;
  bool measured_any = false;
  for (size_t i = 0; i < specs.size(); ++i) {
    if (specs[i].has_profile) {  // given by the rails config: keep it
      profiles.push_back(specs[i].profile);
      continue;
    }
    measured_any = true;
    nz_rail* r = rails[i];
    std::vector<double> lat;
    for (uint64_t s : sizes) {
      const uint64_t C = nezha::defaultChunkBytes(s, world, algo);
      const int iters = s <= (1u << 20) ? std::max(cfg.calibrate_iters, 4) : std::max(cfg.calibrate_iters / 4, 2);
      for (int w = 0; w < 2; ++w) nz::railAllreduce(r, ub_in, ub_out, 0, s, C, 0, UINT64_MAX, NZ_F32, 0, -1, r->stream);
      NZ_CUDA(cudaEventRecord(e0, r->stream));
      for (int it = 0; it < iters; ++it)
        nz::railAllreduce(r, ub_in, ub_out, 0, s, C, 0, UINT64_MAX, NZ_F32, 0, -1, r->stream);
      NZ_CUDA(cudaEventRecord(e1, r->stream));
      NZ_CUDA(cudaEventSynchronize(e1));
      float ms = 0;
      NZ_CUDA(cudaEventElapsedTime(&ms, e0, e1));
      lat.push_back(static_cast<double>(ms) * 1000.0 / iters);
    }
    // Ranks agree (max), then the samples are made strictly increasing so
    // RailProfile::validate accepts them (types.cpp:44-51).
    if (world > 1) {
      const auto msgs = nz::exchange(comm, lat.data(), lat.size() * sizeof(double), {});
      for (int rk = 0; rk < world; ++rk) {
        const double* v = reinterpret_cast<const double*>(msgs[rk].data.data());
        for (size_t j = 0; j < lat.size(); ++j) lat[j] = std::max(lat[j], v[j]);
      }
    }
    for (size_t j = 1; j < lat.size(); ++j) lat[j] = std::max(lat[j], lat[j - 1] + 1e-3);
    nezha::RailProfile p = specs[i].profile;
    p.rail_id = specs[i].rail_id;
    p.efficiency_points.clear();
    for (size_t j = 0; j < sizes.size(); ++j) p.efficiency_points.emplace_back(sizes[j], lat[j]);
    // (t_setup, B) from calibrate(); the measured
    // points stay as the interpolation table messageLatency() uses.
    const nezha::CalibratedProfile cal = nezha::calibrate(p.rail_id, p.protocol, p.efficiency_points);
    p.t_setup_us = cal.profile.t_setup_us;
    p.bandwidth_bps = cal.profile.bandwidth_bps;
    profiles.push_back(p);
    specs[i].profile = p;
    specs[i].has_profile = true;
  }
  bal->setProfiles(profiles);
  if (measured_any && specs.size() > 1) calibrateConcurrent(sizes, e0);
  if (cfg.sync_overhead_us < 0 && specs.size() > 1) {
    // Fork/join of every rail on 4 KiB each vs the slowest rail alone.
    const uint64_t s = 4096;
    const int iters = 50;
    double single = 0;
    for (auto& sp : specs) single = std::max(single, sp.profile.messageLatency(s));
    cudaStream_t user = io;
    NZ_CUDA(cudaEventRecord(e0, user));
    for (int it = 0; it < iters; ++it) {
      cudaEvent_t f = event();
      NZ_CUDA(cudaEventRecord(f, user));
      std::vector<cudaEvent_t> ends;
      for (size_t i = 0; i < rails.size(); ++i) {
        NZ_CUDA(cudaStreamWaitEvent(rails[i]->stream, f, 0));
        nz::railAllreduce(rails[i], ub_in, ub_out, s * i, s, 65536, 0, UINT64_MAX, NZ_F32, 0, -1, rails[i]->stream);
        cudaEvent_t e = event();
        NZ_CUDA(cudaEventRecord(e, rails[i]->stream));
        NZ_CUDA(cudaStreamWaitEvent(user, e, 0));
        ends.push_back(e);
      }
      NZ_CUDA(cudaStreamSynchronize(user));
      pool.push_back(f);
      for (auto e : ends) pool.push_back(e);
    }
    NZ_CUDA(cudaEventRecord(e1, user));
    NZ_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    NZ_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    double multi = static_cast<double>(ms) * 1000.0 / iters;
    if (world > 1) {
      const auto msgs = nz::exchange(comm, &multi, sizeof(multi), {});
      for (int rk = 0; rk < world; ++rk) multi = std::max(multi, *reinterpret_cast<const double*>(msgs[rk].data.data()));
    }
    bal->setSyncOverhead(std::max(0.0, multi - single));
  }
  pool.push_back(e0);
  pool.push_back(e1);
}

void nz_engine::calibrateConcurrent(const std::vector<uint64_t>& sizes, cudaEvent_t start) {
  const int world = comm->world;
  const size_t R = specs.size();
  std::vector<std::vector<double>> lat(R);
  std::vector<uint64_t> shares;
  std::vector<cudaEvent_t> ends(R);
  for (auto& e : ends) e = event();
  for (uint64_t S : sizes) {
    const uint64_t share = std::max<uint64_t>((S / R) & ~uint64_t{15}, 16);
    shares.push_back(share);
    const int iters = S <= (1u << 20) ? std::max(cfg.calibrate_iters, 4) : std::max(cfg.calibrate_iters / 4, 2);
    std::vector<double> acc(R, 0.0);
    std::vector<std::pair<int, uint64_t>> segs;
    for (size_t i = 0; i < R; ++i) segs.emplace_back(specs[i].rail_id, share);
    for (int it = 0; it < iters + 1; ++it) {
      NZ_CUDA(cudaEventRecord(start, io));
      auto gates = gatesFor(segs, nullptr);  // the profiles see the same SM arbitration as the ops
      for (size_t i = 0; i < R; ++i) {
        NZ_CUDA(cudaStreamWaitEvent(rails[i]->stream, start, 0));
        const uint64_t C = nezha::defaultChunkBytes(share, world, algo);
        nz::railAllreduce(rails[i], ub_in, ub_out, share * i, share, C, 0, UINT64_MAX, NZ_F32, 0, -1,
                          rails[i]->stream, &gates[i]);
        NZ_CUDA(cudaEventRecord(ends[i], rails[i]->stream));
        NZ_CUDA(cudaStreamWaitEvent(io, ends[i], 0));
      }
      recycleGates();
      NZ_CUDA(cudaStreamSynchronize(io));
      if (it == 0) continue;  // warm-up
      for (size_t i = 0; i < R; ++i) {
        float ms = 0;
        NZ_CUDA(cudaEventElapsedTime(&ms, start, ends[i]));
        acc[i] += static_cast<double>(ms) * 1000.0;
      }
    }
    for (size_t i = 0; i < R; ++i) lat[i].push_back(acc[i] / iters);
  }
  for (auto e : ends) pool.push_back(e);
  std::vector<nezha::RailProfile> conc;
  for (size_t i = 0; i < R; ++i) {
    auto& l = lat[i];
    if (world > 1) {
      const auto msgs = nz::exchange(comm, l.data(), l.size() * sizeof(double), {});
      for (int rk = 0; rk < world; ++rk) {
        const double* v = reinterpret_cast<const double*>(msgs[rk].data.data());
        for (size_t j = 0; j < l.size(); ++j) l[j] = std::max(l[j], v[j]);
      }
    }
    for (size_t j = 1; j < l.size(); ++j) l[j] = std::max(l[j], l[j - 1] + 1e-3);
    nezha::RailProfile p = specs[i].profile;
    p.efficiency_points.clear();
    for (size_t j = 0; j < shares.size(); ++j) {
      if (j && shares[j] <= shares[j - 1]) continue;
      p.efficiency_points.emplace_back(shares[j], l[j]);
    }
    p.t_setup_us = l.front();
    p.bandwidth_bps =
        static_cast<double>(shares.back() - shares.front()) / std::max(1e-9, (l.back() - l.front()) * 1e-6);
    conc.push_back(p);
  }
  bal->setConcurrentProfiles(conc);
}
