// Host-side mirror of the reference's strategy/plugin API: the MgrStrategy
// value types (proj/include/mgrkit/mgr.hpp:55-77, relax.hpp:21-42,
// amg.hpp:14-24, krylov.hpp:14-19) and the JSON schema that selects them
// (proj/src/strategy_json.cpp:75-228). Same keys, same defaults, same
// unknown-key errors, so every shipped proj/strategies/*.json file is a
// valid input as-is.
#pragma once

#include <memory>
#include <optional>
#include <string>
#include <utility>
#include <vector>

namespace mgrx {

enum class Smoother {
  jacobi,
  l1_jacobi,
  hybrid_l1_gs_forward,
  hybrid_l1_gs_backward,
  block_jacobi_exact,
  amg_vcycle,
  dense_lu,
};

struct AmgSpec;

struct SmootherSpec {
  Smoother kind = Smoother::jacobi;
  int sweeps = 1;
  double weight = 1.0;
  std::vector<int> block_sizes;
  std::vector<std::pair<int, int>> partition;
  std::shared_ptr<const AmgSpec> amg;
  bool use_unknown_map = false;
};

struct AmgSpec {
  double strength_theta = 0.25;
  int max_levels = 25;
  int coarse_size = 50;
  SmootherSpec pre{Smoother::hybrid_l1_gs_forward, 1, 1.0, {}, {}, nullptr, false};
  SmootherSpec post{Smoother::hybrid_l1_gs_backward, 1, 1.0, {}, {}, nullptr, false};
};

// ortho: orthogonalisation of the device GMRES (not part of the reference's
// KrylovConfig): kOrthoDefault / kOrthoCgs2 the low-synchronisation lagged
// CGS2 (lowsync.cu), kOrthoMgs the reference's MGS with the conditional
// re-orthogonalisation (proj/src/krylov.cpp:80-101), bitwise parity mode.
constexpr int kOrthoDefault = 0, kOrthoMgs = 1, kOrthoCgs2 = 2;
struct KrylovSpec {
  int restart = 50;
  int max_iters = 500;
  double rel_tol = 1e-7;
  double abs_tol = 0.0;
  int ortho = kOrthoDefault;
};

enum class Interp { ideal, jacobi };
enum class Restrict { injection, jacobi, ideal };
enum class Coarse { dense_lu, amg_vcycle, gmres_inner };

struct LevelSpec {
  std::vector<std::string> f_fields;
  Interp interp = Interp::jacobi;
  Restrict restrict_kind = Restrict::injection;
  SmootherSpec f_relax;
  std::optional<SmootherSpec> global_relax;
  std::optional<std::vector<int>> ff_block_sizes;
};

struct CoarseSpec {
  Coarse kind = Coarse::dense_lu;
  AmgSpec amg;
  int cycles = 1;
  bool use_unknown_map = false;
  KrylovSpec krylov;
};

struct Strategy {
  std::string name;
  std::vector<LevelSpec> levels;
  CoarseSpec coarse;
};

// Throws mgrx::RuntimeError("strategy json: <where>: <msg>") like the reference.
Strategy parse_strategy(const std::string& text);

}  // namespace mgrx
