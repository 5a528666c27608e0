// pulsecell_gpu/cli_device.hpp -- the device path of the reference's `simulate`
// and `bench` commands, header-only, on the reference's own
// types and writers. A maintainer calls these from cli.cpp behind a --device
// flag; nothing else of the CLI changes.
//
//   gpu::simulate       == cli.cpp:45-78 run_simulate's evolution and file
//                          outputs, with the field resident on the device
//                          (gpu::evolve) and the reference's writers
//   gpu::run_benchmark  == bench.cpp:12-66 time_steps / run_benchmark: one
//                          untimed warm-up step(), then steady_clock over
//                          `steps` step() calls on a host Array2 (the drop-in
//                          call, host<->device copies included); one row, the
//                          device
#pragma once

#include <chrono>
#include <ctime>
#include <string>
#include <thread>

#include "pulsecell/bench.hpp"
#include "pulsecell/snapshot_io.hpp"
#include "pulsecell_gpu/adi_stepper.hpp"

namespace pulsecell::gpu {

inline EvolutionResult simulate(const Grid& grid, const LayerMaterials& layers,
                                SourceModel& source, const SourceSpec& timing,
                                const SolverConfig& solver, const RunnerConfig& runner,
                                Real t_end, const std::string& out_dir,
                                const std::string& header, DeviceOptions opt = {}) {
  AdiStepper stepper(grid, layers, source, timing, solver, opt);
  EvolutionResult res = evolve(stepper, timing, make_field(grid, solver.T0), t_end, runner);
  write_trace(res.trace, runner.probes.size(), out_dir + "/trace.csv", header);
  if (!res.detector_periods.empty())
    write_phase_trace(res.detector_periods, timing.t_per, out_dir + "/trace_phases.csv", header);
  auto outputs = [&](const Array2& field, const std::string& stem) {
    write_snapshot(grid, field, stem + ".csv", SnapshotFormat::Csv, header);
    write_snapshot(grid, field, stem + ".vtk", SnapshotFormat::VtkStructured, header);
  };
  if (res.pre_on) outputs(res.pre_on->field, out_dir + "/snapshot_pre_on");
  if (res.post_off) outputs(res.post_off->field, out_dir + "/snapshot_post_off");
  for (size_t k = 0; k < res.at_times.size(); ++k)
    outputs(res.at_times[k].field, out_dir + "/snapshot_t" + std::to_string(k));
  outputs(res.field, out_dir + "/field_final");
  return res;
}

inline BenchReport run_benchmark(const Grid& grid, const LayerMaterials& mats,
                                 SourceModel& source, const SourceSpec& timing,
                                 const SolverConfig& solver_cfg, int steps, DeviceOptions opt = {}) {
  if (steps < 1) throw ConfigError("bench.steps: must be >= 1");
  BenchReport report;
  report.nr = grid.nr();
  report.nz = grid.nz();
  report.hardware_threads = std::max(1u, std::thread::hardware_concurrency());
  {
    const std::time_t now = std::time(nullptr);
    char buf[32];
    std::strftime(buf, sizeof buf, "%Y-%m-%dT%H:%M:%SZ", std::gmtime(&now));
    report.timestamp = buf;
  }
  AdiStepper stepper(grid, mats, source, timing, solver_cfg, opt);
  Array2 field = make_field(grid, solver_cfg.T0);
  Real t = 0;
  t += stepper.step(field, t).tau_used;  // warm-up, untimed
  const auto begin = std::chrono::steady_clock::now();
  for (int k = 0; k < steps; ++k) t += stepper.step(field, t).tau_used;
  const auto end = std::chrono::steady_clock::now();
  BenchRow row;
  row.workers = 1;  // one device
  row.wall_s = std::chrono::duration<Real>(end - begin).count();
  report.rows.push_back(row);
  return report;
}

}  // namespace pulsecell::gpu
