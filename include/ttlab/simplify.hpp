// Drop-in ttlab/simplify.hpp on the B200: simplify(MPS) (/root/reference/proj/include/ttlab/simplify.hpp:182-195),
// combine (:151-179) and simplify(MPSSum) (:198-215), plus the batched extension simplify_batch
// (no reference counterpart).
#pragma once

#include <optional>

#include "ttlab/forms.hpp"
#include "ttlab/gpu.hpp"

namespace ttlab {

inline CanonicalMPS simplify(const MPS& target, const Strategy& strategy = DEFAULT_STRATEGY,
                             std::optional<MPS> guess = std::nullopt) {
  auto t = gpu::upload(target);
  std::optional<gpu::DMps> g;
  if (guess) g.emplace(gpu::upload(*guess));
  const ttg_strategy s = gpu::to_c(strategy);
  ttg_dmps* out = nullptr;
  gpu::check(gpu::ctx(), ttg_simplify(gpu::ctx(), t.h, &s, g ? g->h : nullptr, &out, nullptr));
  gpu::DMps o(out);
  return gpu::canonical_from(o.h, 0);
}

/// Compress a lazy sum (simplify.hpp:198-215); guess defaults to default_guess (:133-144).
inline CanonicalMPS simplify(const MPSSum& target, const Strategy& strategy = DEFAULT_STRATEGY,
                             std::optional<MPS> guess = std::nullopt) {
  gpu::SumArgs a(target);
  std::optional<gpu::DMps> g;
  if (guess) g.emplace(gpu::upload(*guess));
  const ttg_strategy s = gpu::to_c(strategy);
  ttg_dmps* out = nullptr;
  gpu::check(gpu::ctx(), ttg_simplify_sum(gpu::ctx(), a.n(), a.wr.data(), a.wi.data(), a.handles.data(), &s,
                                          g ? g->h : nullptr, &out, nullptr));
  gpu::DMps o(out);
  return gpu::canonical_from(o.h, 0);
}

/// Closest MPS under `strategy` to sum_l weights[l] states[l] (simplify.hpp:151-179).
inline CanonicalMPS combine(const std::vector<cplx>& weights, const std::vector<MPS>& states,
                            const Strategy& strategy = DEFAULT_STRATEGY) {
  if (weights.empty() || weights.size() != states.size())
    throw shape_error("combine: weights and states must be non-empty and match");
  const auto dims = states.front().physical_dimensions();
  for (const auto& s : states)
    if (s.physical_dimensions() != dims) throw shape_error("combine: states must share physical dimensions");
  return simplify(MPSSum(weights, states), strategy);
}

namespace detail {
/// MPO -> MPS with the (out, in) pair fused into one physical index, and back (simplify.hpp:219-237).
inline MPS flatten_mpo(const MPO& op) {
  std::vector<Tensor3> ts;
  for (index_t n = 0; n < op.size(); ++n) ts.push_back(op[n].fuse_physical());
  return MPS(std::move(ts), 0.0);
}
inline MPO unflatten_mpo(const MPS& state, const std::vector<index_t>& out_dims, const std::vector<index_t>& in_dims) {
  std::vector<Tensor4> ts;
  for (index_t n = 0; n < state.size(); ++n)
    ts.push_back(Tensor4::split_physical(state[n], out_dims[static_cast<size_t>(n)], in_dims[static_cast<size_t>(n)]));
  return MPO(std::move(ts));
}
}  // namespace detail

/// Compress an MPO: flatten, simplify the state on the device, unflatten (simplify.hpp:241-245).
inline MPO simplify_mpo(const MPO& op, const Strategy& strategy = DEFAULT_STRATEGY) {
  const CanonicalMPS compact = simplify(detail::flatten_mpo(op), strategy.with_normalize(false));
  return detail::unflatten_mpo(compact, op.out_dimensions(), op.in_dimensions());
}

/// Compress a weighted sum of MPOs the same way (simplify.hpp:248-260).
inline MPO simplify_mpo(const std::vector<cplx>& weights, const std::vector<MPO>& terms,
                        const Strategy& strategy = DEFAULT_STRATEGY) {
  if (weights.empty() || weights.size() != terms.size())
    throw shape_error("simplify_mpo: weights and terms must be non-empty and match");
  std::vector<MPS> flats;
  for (const auto& t : terms) flats.push_back(detail::flatten_mpo(t));
  const CanonicalMPS compact = simplify(MPSSum(weights, flats), strategy.with_normalize(false));
  return detail::unflatten_mpo(compact, terms.front().out_dimensions(), terms.front().in_dimensions());
}

/// Per-chain scalars of a batch, in global chain order (the payload of the one collective of SURVEY.md 8e).
struct BatchStats {
  std::vector<double> norm, error;
  std::vector<int> sweeps;
};

namespace gpu {
/// Communicator of the multi-GPU batched path (one rank per GPU): rank 0 draws the id, the host program
/// ships its TTG_COMM_ID_BYTES to the other ranks (MPI, a file, a socket ...), every rank joins.  The
/// communicator lives in this thread's context.
inline std::vector<char> comm_unique_id() {
  std::vector<char> id(TTG_COMM_ID_BYTES);
  check(ctx(), ttg_comm_unique_id(ctx(), id.data()));
  return id;
}
inline void comm_init(int nranks, int rank, const std::vector<char>& id) {
  if (id.size() != TTG_COMM_ID_BYTES) throw shape_error("comm_init: the id must be TTG_COMM_ID_BYTES long");
  check(ctx(), ttg_comm_init(ctx(), nranks, rank, id.data()));
}
/// Contiguous balanced block [lo, hi) of `total` chains for `rank` of `nranks` (sizes differ by <= 1).
inline std::pair<index_t, index_t> shard_range(index_t total, int nranks, int rank) {
  const index_t base = total / nranks, extra = total % nranks;
  const index_t lo = rank * base + std::min<index_t>(rank, extra);
  return {lo, lo + base + (rank < extra ? 1 : 0)};
}
}  // namespace gpu

/// Batched simplify of independent, identically shaped chains (one device call).  With `all` given, the
/// chains are this rank's shard (gpu::shard_range) of a batch of `total` chains spread over the ranks of
/// the context's communicator (gpu::comm_init; none = a world of one): after the sweeps one all-gather
/// fills `all` with [norm, error, sweeps] of every chain of the batch, in global order, on every rank.
inline std::vector<CanonicalMPS> simplify_batch(const std::vector<MPS>& targets,
                                                const Strategy& strategy = DEFAULT_STRATEGY,
                                                BatchStats* all = nullptr, index_t total = -1) {
  int nranks = 1, rank = 0;
  gpu::check(gpu::ctx(), ttg_comm_info(gpu::ctx(), &nranks, &rank));
  if (total < 0) total = static_cast<index_t>(targets.size()) * nranks;
  if (all) {
    const auto range = gpu::shard_range(total, nranks, rank);
    if (range.second - range.first != static_cast<index_t>(targets.size()))
      throw shape_error("simplify_batch: the local chains are not this rank's shard of the batch");
  }
  std::vector<CanonicalMPS> res;
  std::vector<ttg_report> reps(targets.size());
  if (!targets.empty()) {
    std::vector<const MPS*> ptrs;
    bool real = true;
    for (const auto& m : targets) {
      ptrs.push_back(&m);
      real = real && gpu::all_real(m.tensors());
    }
    auto t = gpu::upload(ptrs, real);
    const ttg_strategy s = gpu::to_c(strategy);
    ttg_dmps* out = nullptr;
    gpu::check(gpu::ctx(), ttg_simplify(gpu::ctx(), t.h, &s, nullptr, &out, reps.data()));
    gpu::DMps o(out);
    for (size_t c = 0; c < targets.size(); ++c) res.push_back(gpu::canonical_from(o.h, static_cast<int>(c)));
  }
  if (all) {
    index_t width = 0;  // rows per rank in the collective: the largest shard, zero padded
    for (int r = 0; r < nranks; ++r) {
      const auto rg = gpu::shard_range(total, nranks, r);
      width = std::max(width, rg.second - rg.first);
    }
    std::vector<double> send(static_cast<size_t>(3 * width), 0.0), recv(static_cast<size_t>(3 * width * nranks), 0.0);
    for (size_t c = 0; c < reps.size(); ++c) {
      send[3 * c] = reps[c].norm;
      send[3 * c + 1] = reps[c].error;
      send[3 * c + 2] = static_cast<double>(reps[c].sweeps);
    }
    gpu::check(gpu::ctx(), ttg_comm_allgather_f64(gpu::ctx(), send.data(), 3 * width, recv.data()));
    all->norm.clear();
    all->error.clear();
    all->sweeps.clear();
    for (int r = 0; r < nranks; ++r) {
      const auto rg = gpu::shard_range(total, nranks, r);
      for (index_t c = 0; c < rg.second - rg.first; ++c) {
        const double* row = recv.data() + 3 * (static_cast<size_t>(r) * width + c);
        all->norm.push_back(row[0]);
        all->error.push_back(row[1]);
        all->sweeps.push_back(static_cast<int>(row[2]));
      }
    }
  }
  return res;
}

}  // namespace ttlab
