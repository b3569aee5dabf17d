// Host side of the drop-in: the reference's case description (the INI-style
// [lattice]/[model]/[tags]/[objective]/[optimizer]/[output] file,
// config.hpp:16-83) parsed and validated from scratch, and the System the
// reference's build_case assembles (config.cpp:302-427): tag map, design
// field (with the reference's mt19937_64 init noise) and objective support.
// Masks and indexing are bit-identical to the reference's by construction;
// tests/test_masks.py checks them against oracle/_ref.
#include "casebuild.h"

#include <algorithm>
#include <charconv>
#include <cmath>
#include <random>
#include <sstream>

namespace lbgpu {

namespace {

std::string trim(const std::string& s) {
  const auto b = s.find_first_not_of(" \t\r");
  if (b == std::string::npos) return "";
  const auto e = s.find_last_not_of(" \t\r");
  return s.substr(b, e - b + 1);
}

struct CfgError {
  std::string msg;
};

[[noreturn]] void fail(const std::string& origin, int line, const std::string& msg) {
  throw CfgError{origin + ":" + std::to_string(line) + ": " + msg};
}

long parse_long(const std::string& v, const std::string& origin, int line, const std::string& key) {
  long out = 0;
  const auto r = std::from_chars(v.data(), v.data() + v.size(), out);
  if (r.ec != std::errc{} || r.ptr != v.data() + v.size())
    fail(origin, line, "value of '" + key + "' is not an integer: '" + v + "'");
  return out;
}

double parse_double(const std::string& v, const std::string& origin, int line,
                    const std::string& key) {
  double out = 0;
  const auto r = std::from_chars(v.data(), v.data() + v.size(), out);
  if (r.ec != std::errc{} || r.ptr != v.data() + v.size())
    fail(origin, line, "value of '" + key + "' is not a number: '" + v + "'");
  return out;
}

bool parse_bool(const std::string& v, const std::string& origin, int line, const std::string& key) {
  if (v == "true" || v == "1" || v == "on") return true;
  if (v == "false" || v == "0" || v == "off") return false;
  fail(origin, line, "value of '" + key + "' is not a boolean: '" + v + "'");
}

// One key of one section (the reference's apply_key, config.cpp:56-125).
void apply(CaseSpec& c, const std::string& sec, const std::string& key, const std::string& val,
           const std::string& origin, int line) {
  auto L = [&] { return parse_long(val, origin, line, key); };
  auto D = [&] { return parse_double(val, origin, line, key); };
  auto B = [&] { return parse_bool(val, origin, line, key); };
  auto unknown = [&] { fail(origin, line, "unknown key '" + key + "' in section [" + sec + "]"); };
  if (sec == "lattice") {
    if (key == "nx") c.nx = int(L());
    else if (key == "ny") c.ny = int(L());
    else if (key == "nz") c.nz = int(L());
    else unknown();
  } else if (sec == "model") {
    if (key == "nu") c.nu = D();
    else if (key == "beta_fluid") c.beta_fluid = D();
    else if (key == "beta_solid") c.beta_solid = D();
    else if (key == "inlet_dp") c.inlet_dp = D();
    else if (key == "u_clamp") c.u_clamp = D();
    else if (key == "collision") c.collision = val;
    else if (key == "precision") c.precision = int(L());
    else if (key == "omega_nonhydro") c.omega_nonhydro = D();
    else if (key == "switch_theta") c.switch_theta = D();
    else if (key == "switch_form") c.switch_form = val;
    else unknown();
  } else if (sec == "tags") {
    if (key == "geometry") c.geometry = val;
    else if (key == "design_x0") c.design_x0 = int(L());
    else if (key == "design_x1") c.design_x1 = int(L());
    else if (key == "heater_x0") c.heater_x0 = int(L());
    else if (key == "heater_x1") c.heater_x1 = int(L());
    else if (key == "inlet_profile") c.inlet_profile = val;
    else if (key == "inlet_T") c.inlet_T = D();
    else unknown();
  } else if (sec == "objective") {
    if (key == "kind") c.objective = val;
    else if (key == "plane_offset") c.plane_offset = int(L());
    else if (key == "penalty_w0") c.penalty_w0 = D();
    else if (key == "penalty_growth") c.penalty_growth = D();
    else if (key == "penalty_interval") c.penalty_interval = L();
    else if (key == "penalty_start") c.penalty_start = L();
    else if (key == "penalty_cap") c.penalty_cap = D();
    else unknown();
  } else if (sec == "optimizer") {
    if (key == "method") c.method = val;
    else if (key == "iterations") c.iterations = L();
    else if (key == "outer_iterations") c.outer_iterations = L();
    else if (key == "zeta") c.zeta = D();
    else if (key == "zeta_stages") c.zeta_stages = val;
    else if (key == "initial_w") c.initial_w = D();
    else if (key == "init_noise") c.init_noise = D();
    else if (key == "seed") c.seed = static_cast<unsigned long>(L());
    else if (key == "primal_tol") c.primal_tol = D();
    else if (key == "adjoint_tol") c.adjoint_tol = D();
    else if (key == "max_inner") c.max_inner = L();
    else if (key == "adjoint_stop") c.adjoint_stop = val;
    else if (key == "adjoint_kernel") c.adjoint_kernel = val;
    else if (key == "adjoint_cache") c.adjoint_cache = val;
    else if (key == "move_limit") c.move_limit = D();
    else if (key == "threshold_points") c.threshold_points = int(L());
    else if (key == "record_interval") c.record_interval = L();
    else if (key == "workers") c.workers = int(L());
    else unknown();
  } else if (sec == "output") {
    if (key == "dir") c.out_dir = val;
    else if (key == "write_vtk") c.write_vtk = B();
    else if (key == "write_csv") c.write_csv = B();
    else unknown();
  } else {
    fail(origin, line, "unknown section [" + sec + "]");
  }
}

bool one_of(const std::string& v, std::initializer_list<const char*> opts) {
  for (const char* o : opts)
    if (v == o) return true;
  return false;
}

long flat(const CaseSpec& c, int x, int y, int z) {
  return x + long(c.nx) * (y + long(c.ny) * z);
}

void validate_case(const CaseSpec& c);

}  // namespace

bool zeta_stages(const CaseSpec& c, std::vector<std::pair<long, double>>& st, std::string& err);

bool parse_case(const std::string& text, const std::string& overrides, CaseSpec& c,
                std::string& err) {
  try {
    c = CaseSpec{};
    std::istringstream in(text);
    std::string raw, section;
    int line = 0;
    const std::string origin = "<text>";
    while (std::getline(in, raw)) {
      ++line;
      const auto hash = raw.find('#');
      if (hash != std::string::npos) raw.erase(hash);
      const std::string s = trim(raw);
      if (s.empty()) continue;
      if (s.front() == '[') {
        if (s.back() != ']') fail(origin, line, "malformed section header '" + s + "'");
        section = trim(s.substr(1, s.size() - 2));
        continue;
      }
      const auto eq = s.find('=');
      if (eq == std::string::npos) fail(origin, line, "expected key = value, got '" + s + "'");
      const std::string key = trim(s.substr(0, eq));
      const std::string val = trim(s.substr(eq + 1));
      if (key.empty()) fail(origin, line, "empty key");
      if (section.empty()) fail(origin, line, "key '" + key + "' appears before any section");
      apply(c, section, key, val, origin, line);
    }
    std::istringstream ov(overrides);
    while (std::getline(ov, raw)) {
      if (trim(raw).empty()) continue;
      const auto eq = raw.find('=');
      if (eq == std::string::npos) throw CfgError{"override must look like section.key=value: '" + raw + "'"};
      const std::string dotted = trim(raw.substr(0, eq));
      const auto dot = dotted.find('.');
      if (dot == std::string::npos)
        throw CfgError{"override key must look like section.key: '" + dotted + "'"};
      apply(c, dotted.substr(0, dot), dotted.substr(dot + 1), trim(raw.substr(eq + 1)),
            "<override>", 0);
    }
    validate_case(c);
    return true;
  } catch (const CfgError& e) {
    err = e.msg;
    return false;
  }
}

// CaseConfig::validate (config.cpp:241-300), the invariants the hot path and
// its builders rely on.
namespace {
void validate_case(const CaseSpec& c) {
  auto bad = [](const std::string& m) { throw CfgError{m}; };
  if (c.nx < 1 || c.ny < 1 || c.nz < 1) bad("lattice extents must be positive");
  if (!one_of(c.geometry, {"channel", "periodic"})) bad("geometry must be channel or periodic");
  if (c.geometry == "channel" && (c.nx < 3 || c.ny < 3))
    bad("channel geometry needs nx >= 3 and ny >= 3");
  if (c.geometry == "channel" && c.nz != 1 && c.nz < 3) bad("3D channel geometry needs nz >= 3");
  if (!(c.nu > 0)) bad("nu must be positive");
  if (c.beta_fluid < 0 || c.beta_solid < 0) bad("diffusivities must be non-negative");
  if (!(c.u_clamp > 0)) bad("u_clamp must be positive");
  if (!one_of(c.collision, {"fmrt", "bgk"})) bad("collision must be fmrt or bgk");
  if (c.precision != 32 && c.precision != 64) bad("precision must be 32 or 64");
  if (!(c.switch_theta > 0)) bad("switch_theta must be positive");
  if (!one_of(c.switch_form, {"solid_power", "fluid_power"}))
    bad("switch_form must be solid_power or fluid_power");
  auto span_ok = [&](int a, int b, int hi) { return a >= 0 && a <= b && b < hi; };
  if (!(c.design_x0 == -1 && c.design_x1 == -1) && !span_ok(c.design_x0, c.design_x1, c.nx))
    bad("design span must satisfy 0 <= design_x0 <= design_x1 < nx (or both -1)");
  if (!(c.heater_x0 == -1 && c.heater_x1 == -1)) {
    if (!span_ok(c.heater_x0, c.heater_x1, c.nx))
      bad("heater span must satisfy 0 <= heater_x0 <= heater_x1 < nx (or both -1)");
    if (c.objective != "heatflux") bad("a heater is only meaningful for the heatflux objective");
    if (c.geometry != "channel") bad("a heater needs channel geometry");
    if (c.nz > 1 && c.heater_x1 - c.heater_x0 + 1 > c.nz)
      bad("heater plate is wider than the z extent");
  }
  if (!one_of(c.inlet_profile, {"uniform", "split"})) bad("inlet_profile must be uniform or split");
  if (!std::isfinite(c.inlet_T)) bad("inlet_T must be finite");
  if (!one_of(c.objective, {"mixing", "heatflux", "synthetic"}))
    bad("objective kind must be mixing, heatflux or synthetic");
  if (c.plane_offset < 0 || c.plane_offset > c.nx - 1)
    bad("plane_offset must lie inside the lattice");
  if (c.penalty_w0 < 0) bad("penalty weight must be non-negative");
  if (c.penalty_w0 > 0 && !(c.penalty_growth > 1.0)) bad("penalty growth factor must exceed 1");
  if (c.penalty_interval < 1) bad("penalty interval must be at least 1");
  if (c.penalty_start < 0) bad("penalty start must be non-negative");
  if (c.penalty_cap < 0) bad("penalty cap must be non-negative");
  if (!one_of(c.method, {"none", "oneshot", "mma"})) bad("method must be none, oneshot or mma");
  if (c.iterations < 0) bad("iterations must be non-negative");
  if (c.outer_iterations < 0) bad("outer_iterations must be non-negative");
  if (c.zeta < 0) bad("zeta must be non-negative");
  {
    std::vector<std::pair<long, double>> st;
    std::string zerr;
    if (!zeta_stages(c, st, zerr)) bad(zerr);
  }
  if (c.initial_w < 0 || c.initial_w > 1) bad("initial_w must lie in [0,1]");
  if (c.init_noise < 0) bad("init_noise must be non-negative");
  if (!(c.primal_tol > 0) || !(c.adjoint_tol > 0)) bad("tolerances must be positive");
  if (c.max_inner < 1) bad("max_inner must be at least 1");
  if (!one_of(c.adjoint_stop, {"match", "tol"})) bad("adjoint_stop must be match or tol");
  if (!one_of(c.adjoint_kernel, {"analytic", "dual"})) bad("adjoint_kernel must be analytic or dual");
  if (!one_of(c.adjoint_cache, {"off", "on"})) bad("adjoint_cache must be off or on");
  if (c.adjoint_cache == "on" && c.method == "oneshot")
    bad("adjoint_cache cannot be combined with the interleaved one-shot method");
  if (!(c.move_limit > 0) || c.move_limit > 1) bad("move_limit must lie in (0,1]");
  if (c.threshold_points < 2) bad("threshold_points must be at least 2");
  if (c.record_interval < 1) bad("record_interval must be at least 1");
  if (c.workers < 1) bad("workers must be at least 1");
}
}  // namespace

bool set_case_key(CaseSpec& c, const std::string& dotted, const std::string& value,
                  std::string& err) {
  try {
    const auto dot = dotted.find('.');
    if (dot == std::string::npos)
      throw CfgError{"override key must look like section.key: '" + dotted + "'"};
    apply(c, dotted.substr(0, dot), dotted.substr(dot + 1), value, "<override>", 0);
    return true;
  } catch (const CfgError& e) {
    err = e.msg;
    return false;
  }
}

bool check_case(const CaseSpec& c, std::string& err) {
  try {
    validate_case(c);
    return true;
  } catch (const CfgError& e) {
    err = e.msg;
    return false;
  }
}

bool parse_case_text(const std::string& text, const std::string& origin, CaseSpec& c,
                     std::string& err) {
  try {
    c = CaseSpec{};
    std::istringstream in(text);
    std::string raw, section;
    int line = 0;
    while (std::getline(in, raw)) {
      ++line;
      const auto hash = raw.find('#');
      if (hash != std::string::npos) raw.erase(hash);
      const std::string s = trim(raw);
      if (s.empty()) continue;
      if (s.front() == '[') {
        if (s.back() != ']') fail(origin, line, "malformed section header '" + s + "'");
        section = trim(s.substr(1, s.size() - 2));
        continue;
      }
      const auto eq = s.find('=');
      if (eq == std::string::npos) fail(origin, line, "expected key = value, got '" + s + "'");
      const std::string key = trim(s.substr(0, eq));
      const std::string val = trim(s.substr(eq + 1));
      if (key.empty()) fail(origin, line, "empty key");
      if (section.empty()) fail(origin, line, "key '" + key + "' appears before any section");
      apply(c, section, key, val, origin, line);
    }
    return true;
  } catch (const CfgError& e) {
    err = e.msg;
    return false;
  }
}

// CaseConfig::serialize (config.cpp:172-229): every key in canonical order,
// doubles in shortest round-trip form.
std::string serialize_case(const CaseSpec& c) {
  auto D = [](double v) {
    char buf[64];
    const auto r = std::to_chars(buf, buf + sizeof buf, v);
    return std::string(buf, r.ptr);
  };
  std::ostringstream o;
  o << "[lattice]\nnx = " << c.nx << "\nny = " << c.ny << "\nnz = " << c.nz << "\n";
  o << "\n[model]\nnu = " << D(c.nu) << "\nbeta_fluid = " << D(c.beta_fluid)
    << "\nbeta_solid = " << D(c.beta_solid) << "\ninlet_dp = " << D(c.inlet_dp)
    << "\nu_clamp = " << D(c.u_clamp) << "\ncollision = " << c.collision
    << "\nprecision = " << c.precision << "\nomega_nonhydro = " << D(c.omega_nonhydro)
    << "\nswitch_theta = " << D(c.switch_theta) << "\nswitch_form = " << c.switch_form << "\n";
  o << "\n[tags]\ngeometry = " << c.geometry << "\ndesign_x0 = " << c.design_x0
    << "\ndesign_x1 = " << c.design_x1 << "\nheater_x0 = " << c.heater_x0
    << "\nheater_x1 = " << c.heater_x1 << "\ninlet_profile = " << c.inlet_profile
    << "\ninlet_T = " << D(c.inlet_T) << "\n";
  o << "\n[objective]\nkind = " << c.objective << "\nplane_offset = " << c.plane_offset
    << "\npenalty_w0 = " << D(c.penalty_w0) << "\npenalty_growth = " << D(c.penalty_growth)
    << "\npenalty_interval = " << c.penalty_interval << "\npenalty_start = " << c.penalty_start
    << "\npenalty_cap = " << D(c.penalty_cap) << "\n";
  o << "\n[optimizer]\nmethod = " << c.method << "\niterations = " << c.iterations
    << "\nouter_iterations = " << c.outer_iterations << "\nzeta = " << D(c.zeta)
    << "\nzeta_stages = " << c.zeta_stages << "\ninitial_w = " << D(c.initial_w)
    << "\ninit_noise = " << D(c.init_noise) << "\nseed = " << c.seed
    << "\nprimal_tol = " << D(c.primal_tol) << "\nadjoint_tol = " << D(c.adjoint_tol)
    << "\nmax_inner = " << c.max_inner << "\nadjoint_stop = " << c.adjoint_stop
    << "\nadjoint_kernel = " << c.adjoint_kernel << "\nadjoint_cache = " << c.adjoint_cache
    << "\nmove_limit = " << D(c.move_limit) << "\nthreshold_points = " << c.threshold_points
    << "\nrecord_interval = " << c.record_interval << "\nworkers = " << c.workers << "\n";
  o << "\n[output]\ndir = " << c.out_dir << "\nwrite_vtk = " << (c.write_vtk ? "true" : "false")
    << "\nwrite_csv = " << (c.write_csv ? "true" : "false") << "\n";
  return o.str();
}

// parse_zeta_stages (config.cpp:429-452); empty -> one stage {0, zeta}.
bool zeta_stages(const CaseSpec& c, std::vector<std::pair<long, double>>& st, std::string& err) {
  try {
    st.clear();
    if (c.zeta_stages.empty()) {
      st.push_back({0, c.zeta});
      return true;
    }
    std::istringstream in(c.zeta_stages);
    std::string item;
    while (std::getline(in, item, ',')) {
      const auto colon = item.find(':');
      if (colon == std::string::npos)
        throw CfgError{"zeta_stages entries must look like start:value, got '" + item + "'"};
      const long start = parse_long(trim(item.substr(0, colon)), "<zeta_stages>", 0, "zeta_stages");
      const double value =
          parse_double(trim(item.substr(colon + 1)), "<zeta_stages>", 0, "zeta_stages");
      if (value < 0) throw CfgError{"zeta stage values must be non-negative"};
      if (!st.empty() && start <= st.back().first)
        throw CfgError{"zeta stage starts must increase"};
      st.push_back({start, value});
    }
    if (st.empty() || st.front().first != 0)
      throw CfgError{"zeta_stages must begin with a stage at iteration 0"};
    return true;
  } catch (const CfgError& e) {
    err = e.msg;
    return false;
  }
}

bool build_system(const CaseSpec& c, SystemArrays& s, std::string& err) {
  try {
    const long n = long(c.nx) * c.ny * c.nz;
    const bool is3d = c.nz > 1;
    s = SystemArrays{};
    s.tag.assign(n, 0);
    s.bc_T.assign(n, 0.0);
    s.bc_axis.assign(n, 0);
    s.bc_sign.assign(n, 0);
    // build_tags (config.cpp:302-343): walls win, then the x faces, then the
    // heater plate overrides the bottom wall.
    if (c.geometry != "periodic") {
      for (int z = 0; z < c.nz; ++z)
        for (int y = 0; y < c.ny; ++y)
          for (int x = 0; x < c.nx; ++x) {
            const long i = flat(c, x, y, z);
            if (y == 0 || y == c.ny - 1 || (is3d && (z == 0 || z == c.nz - 1))) {
              s.tag[i] = 1;
            } else if (x == 0) {
              s.tag[i] = 2;
              s.bc_axis[i] = 0;
              s.bc_sign[i] = 1;
              s.bc_T[i] = c.inlet_profile == "split" ? (y < c.ny / 2 ? -1.0 : 1.0) : c.inlet_T;
            } else if (x == c.nx - 1) {
              s.tag[i] = 3;
              s.bc_axis[i] = 0;
              s.bc_sign[i] = -1;
            }
          }
      if (c.heater_x0 >= 0) {
        const int width = c.heater_x1 - c.heater_x0 + 1;
        const int z0 = is3d ? (c.nz - width) / 2 : 0;
        const int z1 = is3d ? z0 + width - 1 : 0;
        for (int z = z0; z <= z1; ++z)
          for (int x = c.heater_x0; x <= c.heater_x1; ++x) {
            const long i = flat(c, x, 0, z);
            s.tag[i] = 4;
            s.bc_T[i] = 1.0;
          }
      }
    }
    // build_design (config.cpp:347-371): interior nodes of the x span, w from
    // initial_w plus the reference's deterministic mt19937_64 noise.
    s.mask.assign(n, 0);
    s.w.assign(n, 1.0);
    if (c.design_x0 >= 0)
      for (int z = 0; z < c.nz; ++z)
        for (int y = 0; y < c.ny; ++y)
          for (int x = c.design_x0; x <= c.design_x1; ++x) {
            const long i = flat(c, x, y, z);
            if (s.tag[i] == 0) s.mask[i] = 1;
          }
    std::mt19937_64 rng(c.seed);
    for (long i = 0; i < n; ++i) {
      if (!s.mask[i]) continue;
      double w = c.initial_w;
      if (c.init_noise > 0) {
        const double u = double(rng() >> 11) * 0x1p-53;
        w += c.init_noise * (2.0 * u - 1.0);
      }
      s.w[i] = std::clamp(w, 0.0, 1.0);
    }
    // build_objective (config.cpp:373-395): interior nodes of x = nx-1-offset.
    s.obj_kind = c.objective == "mixing" ? 0 : (c.objective == "heatflux" ? 1 : 2);
    s.flux_axis = 0;
    s.flux_sign = 1;
    const int xp = c.nx - 1 - c.plane_offset;
    for (int z = 0; z < c.nz; ++z)
      for (int y = 0; y < c.ny; ++y) {
        const long i = flat(c, xp, y, z);
        if (s.tag[i] == 0) s.support.push_back(i);
      }
    if (s.support.empty())
      throw CfgError{"objective support plane x = " + std::to_string(xp) + " has no interior nodes"};
    return true;
  } catch (const CfgError& e) {
    err = e.msg;
    return false;
  }
}

// One x-slab of the case (decompose, partition.cpp:9-21): the
// tables of global columns [x0, x0+span) in a local array of nxl columns —
// owned columns at local 0..span-1, the right ghost (global x0+span) at local
// span, the left ghost (global x0-1) at local nxl-1, padding in between (so
// rows stay aligned and the kernels' periodic wrap lands on the ghosts).
// Values are those build_case gives the global lattice, including the
// mt19937_64 design noise (drawn over all design nodes in global order).
bool build_slab(const CaseSpec& c, int x0, int span, int nxl, SystemArrays& s, std::string& err) {
  try {
    if (span < 1 || x0 < 0 || x0 + span > c.nx || nxl < span + 2)
      throw CfgError{"invalid slab geometry"};
    const long n = long(nxl) * c.ny * c.nz;
    const bool is3d = c.nz > 1;
    s = SystemArrays{};
    s.tag.assign(n, 1);
    s.bc_T.assign(n, 0.0);
    s.bc_axis.assign(n, 0);
    s.bc_sign.assign(n, 0);
    s.mask.assign(n, 0);
    s.w.assign(n, 1.0);
    const int hw = c.heater_x1 - c.heater_x0 + 1;
    const int hz0 = is3d ? (c.nz - hw) / 2 : 0, hz1 = is3d ? hz0 + hw - 1 : 0;
    auto gx_of = [&](int lx) {
      if (lx < span) return x0 + lx;
      if (lx == span) return (x0 + span) % c.nx;
      if (lx == nxl - 1) return (x0 - 1 + c.nx) % c.nx;
      return -1;
    };
    for (int z = 0; z < c.nz; ++z)
      for (int y = 0; y < c.ny; ++y)
        for (int lx = 0; lx < nxl; ++lx) {
          const int x = gx_of(lx);
          if (x < 0) continue;
          const long i = lx + long(nxl) * (y + long(c.ny) * z);
          uint8_t t = 0;
          if (c.geometry != "periodic") {
            if (y == 0 || y == c.ny - 1 || (is3d && (z == 0 || z == c.nz - 1))) {
              t = 1;
            } else if (x == 0) {
              t = 2;
              s.bc_sign[i] = 1;
              s.bc_T[i] = c.inlet_profile == "split" ? (y < c.ny / 2 ? -1.0 : 1.0) : c.inlet_T;
            } else if (x == c.nx - 1) {
              t = 3;
              s.bc_sign[i] = -1;
            }
            if (c.heater_x0 >= 0 && y == 0 && x >= c.heater_x0 && x <= c.heater_x1 && z >= hz0 &&
                z <= hz1) {
              t = 4;
              s.bc_T[i] = 1.0;
              s.bc_sign[i] = 0;
            }
          }
          s.tag[i] = t;
        }
    // design: walk every global design node in ascending order, keep ours
    std::mt19937_64 rng(c.seed);
    if (c.design_x0 >= 0)
      for (int z = 0; z < c.nz; ++z)
        for (int y = 0; y < c.ny; ++y)
          for (int x = c.design_x0; x <= c.design_x1; ++x) {
            bool interior = true;
            if (c.geometry != "periodic")
              interior = !(y == 0 || y == c.ny - 1 || (is3d && (z == 0 || z == c.nz - 1)) ||
                           x == 0 || x == c.nx - 1);
            if (!interior) continue;
            double w = c.initial_w;
            if (c.init_noise > 0) {
              const double u = double(rng() >> 11) * 0x1p-53;
              w += c.init_noise * (2.0 * u - 1.0);
            }
            if (x >= x0 && x < x0 + span) {
              const long i = (x - x0) + long(nxl) * (y + long(c.ny) * z);
              s.mask[i] = 1;
              s.w[i] = std::clamp(w, 0.0, 1.0);
            }
          }
    s.obj_kind = c.objective == "mixing" ? 0 : (c.objective == "heatflux" ? 1 : 2);
    s.flux_axis = 0;
    s.flux_sign = 1;
    const int xp = c.nx - 1 - c.plane_offset;
    if (xp >= x0 && xp < x0 + span)
      for (int z = 0; z < c.nz; ++z)
        for (int y = 0; y < c.ny; ++y) {
          const long i = (xp - x0) + long(nxl) * (y + long(c.ny) * z);
          if (s.tag[i] == 0) s.support.push_back(i);
        }
    return true;
  } catch (const CfgError& e) {
    err = e.msg;
    return false;
  }
}

}  // namespace lbgpu
