// Drop-in test: the reference's own AdiStepper (compiled from the reference
// sources) and pulsecell::gpu::AdiStepper (include/pulsecell_gpu) driven
// side by side on the reference's own objects, in one process; exact mode
// must agree bit for bit. Built here by tests/native/Makefile (needs the
// reference headers), run on the GPU box by tests/test_dropin_native.py.
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <unistd.h>
#include <fstream>
#include <sstream>

#include "pulsecell/parallel.hpp"
#include "pulsecell/runner.hpp"
#include "pulsecell/snapshot_io.hpp"
#include "pulsecell/solver.hpp"
#include "pulsecell_gpu/adi_stepper.hpp"
#include "pulsecell_gpu/cli_device.hpp"

namespace {
std::string slurp(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  std::stringstream ss;
  ss << f.rdbuf();
  return ss.str();
}
}  // namespace

using namespace pulsecell;

int main() {
  DomainSpec d;
  d.layer_radii = {1.0e-3, 1.1e-3, 1.4e-3, 1.45e-3};
  d.core_length = 0.022;
  d.outer_length = 0.015;
  d.layer_materials = {"a", "b", "c", "d"};
  d.source_layer = 2;
  GridSpec g;
  g.radial_divisions = {44, 5, 13, 3};
  g.axial_divisions_core = 128;
  g.axial_divisions_outer = 87;
  Grid grid(d, g);
  MaterialSet set;
  const double lam0[4] = {400, 0.1, 5, 1}, alpha[4] = {1.5, 1.0, 2.0, 1.0},
               c0[4] = {1e3, 5e2, 8e2, 6e2};
  for (int m = 0; m < 4; ++m) {
    std::vector<Real> kt, cv, lam;
    for (int k = 4; k <= 300; ++k) {
      kt.push_back(k);
      cv.push_back(c0[m] * std::pow(k / 4.2, 3));
      lam.push_back(lam0[m] * std::pow(k / 4.2, alpha[m]));
    }
    PropertyTable chi;
    if (m == 2) chi = PropertyTable({4.0, 300.0}, {1e-5 * (1 + 0.05 * 4), 1e-5 * (1 + 0.05 * 300)});
    set.add(MaterialTable(d.layer_materials[m], 1.0, PropertyTable(kt, cv), PropertyTable(kt, lam),
                          chi));
  }
  LayerMaterials layers = resolve_layers(set, d.layer_materials);
  SourceSpec timing;
  timing.t_per = 1.0;
  timing.t_src = 0.3;
  timing.t_trs = 0.01;
  timing.I0 = 3.0;
  timing.S_C = d.source_cross_section();
  timing.waveform = Waveform::Rectangular;
  timing.joule_dimensional = true;
  SolverConfig cfg;
  cfg.epsilon = 1e-8;
  cfg.max_iter = 10;
  cfg.tau_transient_divisor = 1000;
  cfg.tau_source_divisor = 300;
  JouleSource src(timing, 2, *layers[2], cfg.range_policy);
  ExecPlan plan;
  plan.workers = 4;
  LinePool pool(plan);
  pulsecell::AdiStepper cpu(grid, layers, src, timing, cfg, pool);
  pulsecell::gpu::AdiStepper gpu(grid, layers, src, timing, cfg, {0});
  Array2 fc = make_field(grid, cfg.T0), fg = make_field(grid, cfg.T0);
  Real t = 0;
  int bad = 0;
  for (int k = 0; k < 40; ++k) {
    const StepResult a = cpu.step(fc, t);
    const StepResult b = gpu.step(fg, t);
    if (a.tau_used != b.tau_used || a.halvings != b.halvings ||
        a.radial.iterations != b.radial.iterations || a.axial.iterations != b.axial.iterations ||
        a.radial.last_delta != b.radial.last_delta || a.axial.last_delta != b.axial.last_delta)
      ++bad;
    t += a.tau_used;
  }
  Index diff = 0;
  for (Index i = 0; i < grid.nr(); ++i)
    for (Index j = 0; j < grid.col_extent(i); ++j)
      if (std::memcmp(&fc(i, j), &fg(i, j), sizeof(Real)) != 0) ++diff;
  // error mapping: max_iter = 1 with a floor above tau0/2 -> TauFloorError
  SolverConfig c1 = cfg;
  c1.max_iter = 1;
  c1.tau_min = 0.9 * initial_tau(0.5, timing, cfg);
  pulsecell::gpu::AdiStepper g1(grid, layers, src, timing, c1, {0});
  bool threw = false;
  Array2 f1 = fg;
  double g_tau = -1, g_floor = -1, g_time = -1, c_tau = -2, c_floor = -2, c_time = -2;
  try {
    g1.step(f1, 0.5);
  } catch (const TauFloorError& e) {
    threw = true;
    g_tau = e.tau();
    g_floor = e.floor();
    g_time = e.time();
  }
  {  // the reference's own exception carries the same tau / floor / time
    pulsecell::AdiStepper c1cpu(grid, layers, src, timing, c1, pool);
    Array2 f1c = fc;
    try {
      c1cpu.step(f1c, 0.5);
    } catch (const TauFloorError& e) {
      c_tau = e.tau();
      c_floor = e.floor();
      c_time = e.time();
    }
  }
  threw = threw && g_tau == c_tau && g_floor == c_floor && g_time == c_time;
  // evolve: the reference's runner on the CPU stepper vs pulsecell::gpu::evolve
  RunnerConfig rc;
  rc.t_end = 0.05;
  rc.probes = {ProbeSpec{0.2e-3, 5e-3}, ProbeSpec{1.2e-3, 12e-3}};
  rc.snapshot_times = {0.0, 0.011, 0.03};
  rc.detector.samples_per_period = 8;
  SolverConfig c2 = cfg;
  c2.tau_transient_divisor = 100;
  c2.tau_source_divisor = 100;
  pulsecell::AdiStepper cpu2(grid, layers, src, timing, c2, pool);
  pulsecell::gpu::AdiStepper gpu2(grid, layers, src, timing, c2, {0});
  const EvolutionResult ec = evolve(cpu2, timing, make_field(grid, cfg.T0), rc.t_end, rc);
  const EvolutionResult eg = pulsecell::gpu::evolve(gpu2, timing, make_field(grid, cfg.T0),
                                                    rc.t_end, rc);
  int ebad = 0;
  if (ec.steps != eg.steps || ec.t != eg.t || ec.reason != eg.reason ||
      ec.trace.size() != eg.trace.size() || ec.at_times.size() != eg.at_times.size() ||
      ec.post_off.has_value() != eg.post_off.has_value())
    ++ebad;
  for (size_t k = 0; ebad == 0 && k < ec.trace.size(); ++k)
    if (ec.trace[k].t != eg.trace[k].t || ec.trace[k].tau != eg.trace[k].tau ||
        ec.trace[k].values != eg.trace[k].values)
      ++ebad;
  auto same = [&](const Array2& a, const Array2& b) {
    for (Index i = 0; i < grid.nr(); ++i)
      for (Index j = 0; j < grid.col_extent(i); ++j)
        if (std::memcmp(&a(i, j), &b(i, j), sizeof(Real)) != 0) return false;
    return true;
  };
  for (size_t k = 0; ebad == 0 && k < ec.at_times.size(); ++k)
    if (ec.at_times[k].t != eg.at_times[k].t || !same(ec.at_times[k].field, eg.at_times[k].field))
      ++ebad;
  if (ebad == 0 && ec.post_off && (ec.post_off->t != eg.post_off->t ||
                                   !same(ec.post_off->field, eg.post_off->field)))
    ++ebad;
  if (ebad == 0 && !same(ec.field, eg.field)) ++ebad;
  // simulate --device (cli_device.hpp): the files of cli.cpp's run_simulate,
  // written by the reference's writers from the CPU evolve above and from
  // gpu::simulate, must be byte-identical
  namespace fs = std::filesystem;
  const fs::path base = fs::temp_directory_path() / ("pcgpu_cli_" + std::to_string(::getpid()));
  const std::string dc = (base / "cpu").string(), dg = (base / "gpu").string();
  fs::create_directories(dc);
  fs::create_directories(dg);
  const std::string header = "# dropin cli test";
  write_trace(ec.trace, rc.probes.size(), dc + "/trace.csv", header);
  if (!ec.detector_periods.empty())
    write_phase_trace(ec.detector_periods, timing.t_per, dc + "/trace_phases.csv", header);
  auto outputs = [&](const Array2& f, const std::string& stem) {
    write_snapshot(grid, f, stem + ".csv", SnapshotFormat::Csv, header);
    write_snapshot(grid, f, stem + ".vtk", SnapshotFormat::VtkStructured, header);
  };
  if (ec.pre_on) outputs(ec.pre_on->field, dc + "/snapshot_pre_on");
  if (ec.post_off) outputs(ec.post_off->field, dc + "/snapshot_post_off");
  for (size_t k = 0; k < ec.at_times.size(); ++k)
    outputs(ec.at_times[k].field, dc + "/snapshot_t" + std::to_string(k));
  outputs(ec.field, dc + "/field_final");
  pulsecell::gpu::simulate(grid, layers, src, timing, c2, rc, rc.t_end, dg, header, {0});
  int files = 0, fbad = 0;
  for (const auto& e : fs::directory_iterator(dc)) {
    ++files;
    const fs::path other = fs::path(dg) / e.path().filename();
    if (!fs::exists(other) || slurp(e.path().string()) != slurp(other.string())) ++fbad;
  }
  for (const auto& e : fs::directory_iterator(dg))
    if (!fs::exists(fs::path(dc) / e.path().filename())) ++fbad;
  fs::remove_all(base);
  // bench --device: the timing loop of bench.cpp on the GPU stepper
  const BenchReport br = pulsecell::gpu::run_benchmark(grid, layers, src, timing, cfg, 3, {0});
  const bool bench_ok = br.rows.size() == 1 && br.rows[0].wall_s > 0 && br.nr == grid.nr();
  std::printf("dropin: steps with mismatching results %d, masked cells differing %ld, "
              "TauFloorError mapped %s, evolve (%ld steps, %zu snapshots) %s, "
              "simulate --device files %d differing %d, bench --device %s\n", bad,
              static_cast<long>(diff), threw ? "yes" : "no", ec.steps, ec.at_times.size(),
              ebad ? "DIFFERS" : "identical", files, fbad, bench_ok ? "ok" : "FAILED");
  return (bad == 0 && diff == 0 && threw && ebad == 0 && files > 0 && fbad == 0 && bench_ok)
             ? 0
             : 1;
}
