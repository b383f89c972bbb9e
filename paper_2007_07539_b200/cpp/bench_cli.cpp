// mpmg_bench -- the sweep harness SPEC.md describes (module bench_cli,
// SPEC.md:432-485) and the reference never shipped.
// It is built on the drop-in C++ API (include/mpmg/*.hpp), so every solve is
// the device path a reference caller would get: build_problem ->
// MgHierarchy::build -> ir_solve.
//
//   mpmg_bench --dim 2 --k 1,20,400 --nodes 257,513,1025 --variant d_mg,h_mg \
//              --out sweep.csv [--plot-dir DIR]
//
// Output: one CsvRow per (run x repetition) with the header SPEC.md:441-444
// names exactly, a Table-3-shaped summary (variant x k, mean iterations over
// the grid sizes, one decimal) on stdout, and optionally one
// (iteration, residual) plot-data file per run (emit_convergence_plotdata,
// SPEC.md:455-462). Exit codes: 0 all converged, 1 a run did not
// converge or failed (its row is still written), 2 usage error.
#include <cerrno>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <optional>
#include <sstream>
#include <tuple>
#include <string>
#include <vector>

#include "mpmg/errors.hpp"
#include "mpmg/ir_solver.hpp"
#include "mpmg/kernels.hpp"
#include "mpmg/mesh_fem.hpp"
#include "mpmg/multigrid.hpp"

using namespace mpmg;

namespace {

struct RunSpec {
  std::vector<int> dims{2};
  std::vector<int> ks{1};
  std::vector<int> nodes{65};
  int levels = 0;  // 0: as deep as the grid allows (base of 3 nodes)
  std::vector<MgVariant> variants{MgVariant::D_MG};
  std::uint64_t seed = 0;
  int reps = 1;
  std::string out = "mpmg_sweep.csv";
  std::string plot_dir;
  double tol_outer = 1e-9;  // absolute, ir_solver.hpp:16
  bool tol_relative = false;
  double tol_base = 1e-4;
  int nu1 = 3, nu2 = 3;
  double omega = 2.0 / 3.0;
  Fp16Accum acc = Fp16Accum::FP16;
  bool ftz = true;
  bool validate = false;
  bool random_init = false;
  int max_iterations = 100;
};

[[noreturn]] void usage(const std::string& why) {
  std::fprintf(stderr,
               "mpmg_bench: %s\n"
               "usage: mpmg_bench [--dim D[,D]] [--k K[,K..]] [--nodes N[,N..]] [--levels L]\n"
               "                  [--variant d_mg|h_mg|dsh_mg|hsd_mg[,..]] [--seed S] [--reps R] [--out FILE]\n"
               "                  [--tol-outer T] [--tol-relative] [--tol-base T] [--nu1 N] [--nu2 N] [--omega W]\n"
               "                  [--fp16-accum fp16|fp32] [--no-ftz] [--validate] [--random-init]\n"
               "                  [--max-iterations N] [--plot-dir DIR]\n",
               why.c_str());
  std::exit(2);
}

long parse_int(const std::string& s, const char* flag) {
  char* end = nullptr;
  errno = 0;
  const long v = std::strtol(s.c_str(), &end, 10);
  if (errno || end == s.c_str() || *end) usage(std::string("bad integer for ") + flag + ": '" + s + "'");
  return v;
}
double parse_double(const std::string& s, const char* flag) {
  char* end = nullptr;
  errno = 0;
  const double v = std::strtod(s.c_str(), &end);
  if (errno || end == s.c_str() || *end) usage(std::string("bad number for ") + flag + ": '" + s + "'");
  return v;
}
std::vector<std::string> split(const std::string& s) {
  std::vector<std::string> out;
  std::stringstream ss(s);
  std::string item;
  while (std::getline(ss, item, ','))
    if (!item.empty()) out.push_back(item);
  return out;
}

RunSpec parse_args(int argc, char** argv) {
  RunSpec r;
  for (int i = 1; i < argc; ++i) {
    const std::string a = argv[i];
    auto value = [&](const char* flag) -> std::string {
      if (i + 1 >= argc) usage(std::string("missing value for ") + flag);
      return argv[++i];
    };
    auto int_list = [&](const char* flag) {
      std::vector<int> v;
      for (const auto& s : split(value(flag))) v.push_back(static_cast<int>(parse_int(s, flag)));
      if (v.empty()) usage(std::string("empty list for ") + flag);
      return v;
    };
    if (a == "--dim") r.dims = int_list("--dim");
    else if (a == "--k") r.ks = int_list("--k");
    else if (a == "--nodes") r.nodes = int_list("--nodes");
    else if (a == "--levels") r.levels = static_cast<int>(parse_int(value("--levels"), "--levels"));
    else if (a == "--variant") {
      r.variants.clear();
      for (const auto& s : split(value("--variant"))) {
        auto v = parse_variant(s);
        if (!v) usage("unknown variant '" + s + "'");
        r.variants.push_back(*v);
      }
      if (r.variants.empty()) usage("empty --variant list");
    } else if (a == "--seed") r.seed = static_cast<std::uint64_t>(parse_int(value("--seed"), "--seed"));
    else if (a == "--reps") r.reps = static_cast<int>(parse_int(value("--reps"), "--reps"));
    else if (a == "--out") r.out = value("--out");
    else if (a == "--plot-dir") r.plot_dir = value("--plot-dir");
    else if (a == "--tol-outer") r.tol_outer = parse_double(value("--tol-outer"), "--tol-outer");
    else if (a == "--tol-relative") r.tol_relative = true;
    else if (a == "--tol-base") r.tol_base = parse_double(value("--tol-base"), "--tol-base");
    else if (a == "--nu1") r.nu1 = static_cast<int>(parse_int(value("--nu1"), "--nu1"));
    else if (a == "--nu2") r.nu2 = static_cast<int>(parse_int(value("--nu2"), "--nu2"));
    else if (a == "--omega") r.omega = parse_double(value("--omega"), "--omega");
    else if (a == "--fp16-accum") {
      const std::string v = value("--fp16-accum");
      if (v == "fp16") r.acc = Fp16Accum::FP16;
      else if (v == "fp32") r.acc = Fp16Accum::FP32;
      else usage("--fp16-accum takes fp16 or fp32");
    } else if (a == "--no-ftz") r.ftz = false;
    else if (a == "--validate") r.validate = true;
    else if (a == "--random-init") r.random_init = true;
    else if (a == "--max-iterations") r.max_iterations = static_cast<int>(parse_int(value("--max-iterations"), a.c_str()));
    else if (a == "-h" || a == "--help") usage("help");
    else usage("unknown flag '" + a + "'");
  }
  if (r.reps < 1) usage("--reps must be >= 1");
  if (r.nu1 < 0 || r.nu2 < 0) usage("--nu1/--nu2 must be >= 0");
  if (!(r.tol_outer > 0.0)) usage("--tol-outer must be positive");
  for (int d : r.dims)
    if (d != 2 && d != 3) usage("--dim must be 2 or 3");
  for (int n : r.nodes) {  // RunSpec invariant: every size compatible with the levels
    if (n < 3) usage("--nodes entries must be >= 3");
    const int L = r.levels;
    if (L > 0 && ((n - 1) % (1 << (L - 1)) != 0 || ((n - 1) >> (L - 1)) + 1 < 3))
      usage("nodes " + std::to_string(n) + " incompatible with --levels " + std::to_string(L));
  }
  return r;
}

int max_levels(int nodes) {  // deepest hierarchy with a base of >= 3 nodes
  int L = 1;
  while ((nodes - 1) % (1 << L) == 0 && ((nodes - 1) >> L) + 1 >= 3) ++L;
  return L;
}

std::string fmt(double v) {
  char buf[64];
  std::snprintf(buf, sizeof buf, "%.17g", v);
  return buf;
}

// emit_convergence_plotdata: header, then one
// (iteration, residual) row per history entry.
void emit_plotdata(const std::string& path, const SolveReport& rep) {
  std::ofstream f(path);
  f << "# iteration residual_norm\n";
  for (std::size_t i = 0; i < rep.residual_history.size(); ++i) f << i << ' ' << fmt(rep.residual_history[i]) << '\n';
}

}  // namespace

int main(int argc, char** argv) {
  const RunSpec spec = parse_args(argc, argv);
  std::ofstream csv(spec.out);
  if (!csv) usage("cannot open --out " + spec.out);
  csv << "dim,k,nodes_per_dim,variant,iterations,final_residual,l2_error_vs_exact,value_bytes_moved,wall_time_s,seed\n";
  csv.flush();

  // (variant, dim, k) -> (sum of iterations, runs) for the Table-3 summary
  std::map<std::tuple<int, int, int>, std::pair<long, long>> table;
  bool all_converged = true;

  for (int dim : spec.dims)
    for (int k : spec.ks)
      for (int nodes : spec.nodes) {
        const int L = spec.levels > 0 ? spec.levels : max_levels(nodes);
        const ProblemSpec ps{dim, k, nodes, L};
        std::optional<Problem> prob;
        try {
          prob = build_problem(ps);
        } catch (const std::exception& e) {
          std::fprintf(stderr, "mpmg_bench: build_problem(dim=%d k=%d n=%d L=%d) failed: %s\n", dim, k, nodes, L,
                       e.what());
          for (MgVariant v : spec.variants)
            for (int rep = 0; rep < spec.reps; ++rep)
              csv << dim << ',' << k << ',' << nodes << ',' << variant_name(v) << ",-1,nan,nan,0,0," << spec.seed
                  << '\n';
          csv.flush();
          all_converged = false;
          continue;
        }
        const ArithmeticPolicy policy{spec.ftz, true};
        ExecContext ctx;
        ctx.policy = policy;
        ctx.fp16_accumulation = spec.acc;
        ctx.validate = spec.validate;
        const double bnorm = norm2_fp64(prob->b, ctx);
        for (MgVariant v : spec.variants)
          for (int rep = 0; rep < spec.reps; ++rep) {
            std::string row;
            try {
              BaseSolverConfig base;
              base.tolerance = spec.tol_base;
              MgHierarchy h = MgHierarchy::build(ps, v, SmootherConfig{spec.nu1, spec.nu2, spec.omega}, base, policy);
              IrConfig cfg;
              cfg.outer_tolerance = spec.tol_relative ? spec.tol_outer * bnorm : spec.tol_outer;
              cfg.max_outer_iterations = spec.max_iterations;
              cfg.seed = spec.seed;
              cfg.initial_guess =
                  spec.random_init ? IrConfig::InitialGuess::SeededRandom01 : IrConfig::InitialGuess::Zeros;
              IrResult res = ir_solve(prob->A, prob->b, h, cfg, ctx);
              const SolveReport& r = res.report;
              const double err = nodal_l2_error(res.u, prob->u_exact, prob->grid);
              std::ostringstream o;
              o << dim << ',' << k << ',' << nodes << ',' << variant_name(v) << ',' << r.iterations << ','
                << fmt(r.final_residual) << ',' << fmt(err) << ',' << r.total_traffic().value_bytes() << ','
                << fmt(r.wall_time_s) << ',' << spec.seed << '\n';
              row = o.str();
              if (!r.converged) all_converged = false;
              auto& cell = table[{static_cast<int>(v), dim, k}];
              cell.first += r.iterations;
              cell.second += 1;
              if (!spec.plot_dir.empty())
                emit_plotdata(spec.plot_dir + "/" + std::to_string(dim) + "d_k" + std::to_string(k) + "_n" +
                                  std::to_string(nodes) + "_" + std::string(variant_name(v)) + "_rep" +
                                  std::to_string(rep) + ".dat",
                              r);
            } catch (const DivergedError& e) {
              std::fprintf(stderr, "mpmg_bench: %s diverged: %s\n", std::string(variant_name(v)).c_str(), e.what());
              row = std::to_string(dim) + ',' + std::to_string(k) + ',' + std::to_string(nodes) + ',' +
                    std::string(variant_name(v)) + ",-1,inf,nan,0,0," + std::to_string(spec.seed) + '\n';
              all_converged = false;
            } catch (const std::exception& e) {
              std::fprintf(stderr, "mpmg_bench: %s failed: %s\n", std::string(variant_name(v)).c_str(), e.what());
              row = std::to_string(dim) + ',' + std::to_string(k) + ',' + std::to_string(nodes) + ',' +
                    std::string(variant_name(v)) + ",-1,nan,nan,0,0," + std::to_string(spec.seed) + '\n';
              all_converged = false;
            }
            csv << row;
            csv.flush();  // partial CSV survives a later failure
          }
      }

  // Table-3-shaped summary: variant x k, mean iterations over the grid sizes.
  // Integer-safe rounding to one decimal: round(10 * sum / n) / 10.
  for (int dim : spec.dims) {
    std::printf("\n%dD: mean iterations over nodes {", dim);
    for (std::size_t i = 0; i < spec.nodes.size(); ++i) std::printf("%s%d", i ? "," : "", spec.nodes[i]);
    std::printf("}\n%-8s", "variant");
    for (int k : spec.ks) std::printf("  k=%-6d", k);
    std::printf("\n");
    for (MgVariant v : spec.variants) {
      std::printf("%-8s", std::string(variant_name(v)).c_str());
      for (int k : spec.ks) {
        auto it = table.find({static_cast<int>(v), dim, k});
        if (it == table.end() || it->second.second == 0) {
          std::printf("  %-8s", "-");
          continue;
        }
        const long s = it->second.first, n = it->second.second;
        const long tenths = (20 * s + n) / (2 * n);
        std::printf("  %ld.%ld     ", tenths / 10, tenths % 10);
      }
      std::printf("\n");
    }
  }
  return all_converged ? 0 : 1;
}
