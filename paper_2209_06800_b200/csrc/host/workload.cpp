// Neighbor-partition / warp-mapping builder (see include/mgg/workload.hpp).
#include "mgg/workload.hpp"

#include <algorithm>
#include <atomic>

#include <nlohmann/json.hpp>

#include "mgg/errors.hpp"
#include "parallel.hpp"

namespace mgg {

namespace {

void require_ps(std::uint32_t ps) {
  if (ps < 1 || ps > kMaxPs)
    throw ConfigError("partition_neighbors: ps=" + std::to_string(ps) +
                      " outside [1," + std::to_string(kMaxPs) + "]");
}
void require_dist(std::uint32_t dist) {
  if (dist < 1 || dist > kMaxDist)
    throw ConfigError("interleave: dist=" + std::to_string(dist) +
                      " outside [1," + std::to_string(kMaxDist) + "]");
}
void require_wpb(std::uint32_t wpb) {
  if (wpb < 1 || wpb > kMaxWpb)
    throw ConfigError("map_to_blocks: wpb=" + std::to_string(wpb) +
                      " outside [1," + std::to_string(kMaxWpb) + "]");
}

// Owner lookup over the ascending NE ranges: index of the first range whose
// ub exceeds id (translate's rule, empty ranges skipped).
struct OwnerIndex {
  std::vector<NodeId> ubs;
  explicit OwnerIndex(const NePlacement& p) {
    for (const auto& r : p.ranges) ubs.push_back(r.ub);
  }
  std::uint32_t operator()(NodeId id) const {
    return static_cast<std::uint32_t>(
        std::upper_bound(ubs.begin(), ubs.end(), id) - ubs.begin());
  }
};

void append_group(WarpWorkload& w, PartKind kind, std::uint64_t begin,
                  std::uint64_t total, std::uint32_t dist) {
  const std::uint64_t end = std::min<std::uint64_t>(begin + dist, total);
  for (std::uint64_t i = begin; i < end; ++i)
    w.tasks.push_back({kind, static_cast<std::uint32_t>(i)});
}

std::vector<BlockAssignment> tile_blocks(std::uint64_t warps, std::uint32_t wpb) {
  std::vector<BlockAssignment> b;
  b.reserve((warps + wpb - 1) / wpb);
  for (std::uint64_t f = 0; f < warps; f += wpb)
    b.push_back({static_cast<std::uint32_t>(f),
                 static_cast<std::uint32_t>(std::min<std::uint64_t>(wpb, warps - f))});
  return b;
}

}  // namespace

LocalRemoteSplit split_local_remote(const CsrGraph& g, const WorkloadSplit& split,
                                    const NePlacement& placement,
                                    std::uint32_t gpu_id) {
  if (gpu_id >= split.num_gpus)
    throw InputError("split_local_remote: gpu_id out of range");
  if (split.num_nodes != g.num_nodes || placement.num_nodes != g.num_nodes)
    throw InputError("split_local_remote: inconsistent node counts");
  const NodeRange chunk = split.chunk_ranges[gpu_id];
  const OwnerIndex owner(placement);
  LocalRemoteSplit out;
  out.gpu_id = gpu_id;
  out.first_target = chunk.lb;
  const std::uint64_t rows = chunk.size();
  for (CsrGraph* c : {&out.local_csr, &out.remote_csr}) {
    c->num_nodes = rows;
    c->row_ptr.assign(rows + 1, 0);
  }
  for (std::uint64_t r = 0; r < rows; ++r) {
    for (NodeId nb : g.neighbors(chunk.lb + r))
      (owner(nb) == gpu_id ? out.local_csr : out.remote_csr).col_idx.push_back(nb);
    out.local_csr.row_ptr[r + 1] = out.local_csr.col_idx.size();
    out.remote_csr.row_ptr[r + 1] = out.remote_csr.col_idx.size();
  }
  return out;
}

std::vector<NeighborPartition> partition_neighbors(const CsrGraph& csr,
                                                   NodeId first_target,
                                                   PartKind kind,
                                                   std::uint32_t ps) {
  require_ps(ps);
  std::vector<NeighborPartition> parts;
  for (std::uint64_t r = 0; r < csr.num_nodes; ++r) {
    const auto nb = csr.neighbors(r);
    for (std::size_t off = 0; off < nb.size(); off += ps) {
      const std::size_t len = std::min<std::size_t>(ps, nb.size() - off);
      parts.push_back({first_target + r, kind,
                       std::vector<NodeId>(nb.begin() + off, nb.begin() + off + len)});
    }
  }
  return parts;
}

std::vector<WarpWorkload> interleave(const std::vector<NeighborPartition>& local_parts,
                                     const std::vector<NeighborPartition>& remote_parts,
                                     std::uint32_t dist) {
  require_dist(dist);
  const std::uint64_t nl = local_parts.size(), nr = remote_parts.size();
  const std::uint64_t nw = (std::max(nl, nr) + dist - 1) / dist;
  std::vector<WarpWorkload> warps(nw);
  for (std::uint64_t w = 0; w < nw; ++w) {
    warps[w].warp_id = static_cast<std::uint32_t>(w);
    if (w * dist < nl) append_group(warps[w], PartKind::local, w * dist, nl, dist);
    if (w * dist < nr) append_group(warps[w], PartKind::remote, w * dist, nr, dist);
  }
  return warps;
}

std::vector<WarpWorkload> map_segregated(
    const std::vector<NeighborPartition>& local_parts,
    const std::vector<NeighborPartition>& remote_parts, std::uint32_t dist) {
  require_dist(dist);
  std::vector<WarpWorkload> warps;
  for (PartKind kind : {PartKind::local, PartKind::remote}) {
    const std::uint64_t n =
        kind == PartKind::local ? local_parts.size() : remote_parts.size();
    for (std::uint64_t b = 0; b < n; b += dist) {
      WarpWorkload w;
      w.warp_id = static_cast<std::uint32_t>(warps.size());
      append_group(w, kind, b, n, dist);
      warps.push_back(std::move(w));
    }
  }
  return warps;
}

KernelLaunchPlan map_to_blocks(std::vector<NeighborPartition> local_parts,
                               std::vector<NeighborPartition> remote_parts,
                               std::vector<WarpWorkload> warps,
                               const KernelConfig& cfg, std::uint64_t dim) {
  require_wpb(cfg.wpb);
  KernelLaunchPlan plan;
  plan.cfg = cfg;
  plan.dim = dim;
  plan.local_parts = std::move(local_parts);
  plan.remote_parts = std::move(remote_parts);
  plan.warps = std::move(warps);
  plan.smem_bytes_per_block = smem(cfg, dim);
  plan.blocks = tile_blocks(plan.warps.size(), cfg.wpb);
  return plan;
}

KernelLaunchPlan build_launch_plan(const LocalRemoteSplit& lr,
                                   const KernelConfig& cfg, std::uint64_t dim,
                                   MappingMode mapping, Granularity granularity) {
  std::vector<NeighborPartition> local, remote;
  if (granularity == Granularity::partitioned) {
    local = partition_neighbors(lr.local_csr, lr.first_target, PartKind::local, cfg.ps);
    remote = partition_neighbors(lr.remote_csr, lr.first_target, PartKind::remote, cfg.ps);
  } else {
    auto whole = [&](const CsrGraph& csr, PartKind kind) {
      std::vector<NeighborPartition> parts;
      for (std::uint64_t r = 0; r < csr.num_nodes; ++r) {
        const auto nb = csr.neighbors(r);
        if (!nb.empty())
          parts.push_back({lr.first_target + r, kind,
                           std::vector<NodeId>(nb.begin(), nb.end())});
      }
      return parts;
    };
    local = whole(lr.local_csr, PartKind::local);
    remote = whole(lr.remote_csr, PartKind::remote);
  }
  auto warps = mapping == MappingMode::interleaved
                   ? interleave(local, remote, cfg.dist)
                   : map_segregated(local, remote, cfg.dist);
  return map_to_blocks(std::move(local), std::move(remote), std::move(warps), cfg, dim);
}

void validate_plan(const KernelLaunchPlan& plan) {
  std::vector<std::uint8_t> seen[2] = {
      std::vector<std::uint8_t>(plan.local_parts.size(), 0),
      std::vector<std::uint8_t>(plan.remote_parts.size(), 0)};
  for (const WarpWorkload& w : plan.warps)
    for (const WarpTask& t : w.tasks) {
      auto& s = seen[t.kind == PartKind::local ? 0 : 1];
      if (t.index >= s.size())
        throw IntegrityError("plan: warp " + std::to_string(w.warp_id) +
                             " references unknown partition " +
                             std::to_string(t.index));
      if (s[t.index]++)
        throw IntegrityError("plan: partition " + std::to_string(t.index) +
                             " assigned to more than one warp");
    }
  const char* names[2] = {"local", "remote"};
  for (int k = 0; k < 2; ++k)
    for (std::size_t i = 0; i < seen[k].size(); ++i)
      if (!seen[k][i])
        throw IntegrityError(std::string("plan: ") + names[k] + " partition " +
                             std::to_string(i) + " not assigned to any warp");
  std::uint64_t covered = 0;
  for (const BlockAssignment& b : plan.blocks) {
    if (b.first_warp != covered || b.warp_count == 0 || b.warp_count > plan.cfg.wpb)
      throw IntegrityError("plan: blocks must tile warps in order");
    covered += b.warp_count;
  }
  if (covered != plan.warps.size())
    throw IntegrityError("plan: blocks do not cover all warps");
}

std::string plan_to_json(const KernelLaunchPlan& plan) {
  auto parts_json = [](const std::vector<NeighborPartition>& ps) {
    nlohmann::json a = nlohmann::json::array();
    for (const auto& p : ps)
      a.push_back({{"target", p.target},
                   {"kind", p.kind == PartKind::local ? "local" : "remote"},
                   {"neighbors", p.neighbors}});
    return a;
  };
  nlohmann::json warps = nlohmann::json::array();
  for (const auto& w : plan.warps) {
    nlohmann::json tasks = nlohmann::json::array();
    for (const auto& t : w.tasks)
      tasks.push_back(nlohmann::json::array(
          {t.kind == PartKind::local ? "local" : "remote", t.index}));
    warps.push_back({{"warp", w.warp_id}, {"tasks", std::move(tasks)}});
  }
  return nlohmann::json{
      {"cfg", {{"ps", plan.cfg.ps}, {"dist", plan.cfg.dist}, {"wpb", plan.cfg.wpb}}},
      {"dim", plan.dim},
      {"smemBytesPerBlock", plan.smem_bytes_per_block},
      {"localParts", parts_json(plan.local_parts)},
      {"remoteParts", parts_json(plan.remote_parts)},
      {"warps", std::move(warps)}}
      .dump();
}

KernelLaunchPlan plan_from_json(const std::string& text) {
  KernelLaunchPlan plan;
  try {
    const auto j = nlohmann::json::parse(text);
    const auto& c = j.at("cfg");
    c.at("ps").get_to(plan.cfg.ps);
    c.at("dist").get_to(plan.cfg.dist);
    c.at("wpb").get_to(plan.cfg.wpb);
    j.at("dim").get_to(plan.dim);
    j.at("smemBytesPerBlock").get_to(plan.smem_bytes_per_block);
    for (const char* key : {"localParts", "remoteParts"}) {
      auto& dst = key[0] == 'l' ? plan.local_parts : plan.remote_parts;
      for (const auto& pj : j.at(key)) {
        NeighborPartition p;
        p.target = pj.at("target").get<NodeId>();
        const std::string k = pj.at("kind").get<std::string>();
        if (k != "local" && k != "remote")
          throw ParseError("plan: unknown partition kind '" + k + "'", 0);
        p.kind = k == "local" ? PartKind::local : PartKind::remote;
        pj.at("neighbors").get_to(p.neighbors);
        dst.push_back(std::move(p));
      }
    }
    for (const auto& wj : j.at("warps")) {
      WarpWorkload w;
      w.warp_id = wj.at("warp").get<std::uint32_t>();
      for (const auto& tj : wj.at("tasks"))
        w.tasks.push_back({tj.at(0).get<std::string>() == "local" ? PartKind::local
                                                                  : PartKind::remote,
                           tj.at(1).get<std::uint32_t>()});
      plan.warps.push_back(std::move(w));
    }
  } catch (const nlohmann::json::exception& e) {
    throw ParseError(std::string("plan: ") + e.what(), 0);
  }
  plan.blocks = tile_blocks(plan.warps.size(), plan.cfg.wpb);
  validate_plan(plan);
  return plan;
}

// ---------------------------------------------------------------------------
// Device form

std::uint64_t FlatPlan::num_warps() const {
  const std::uint64_t nl = local.num_parts(), nr = remote.num_parts();
  if (mapping == MappingMode::interleaved)
    return (std::max(nl, nr) + cfg.dist - 1) / cfg.dist;
  return (nl + cfg.dist - 1) / cfg.dist + (nr + cfg.dist - 1) / cfg.dist;
}

KernelLaunchPlan FlatPlan::expand() const {
  auto unpack = [&](const FlatPartList& l, PartKind kind) {
    std::vector<NeighborPartition> parts(l.num_parts());
    for (std::uint64_t i = 0; i < parts.size(); ++i) {
      parts[i].target = first_target + static_cast<NodeId>(l.meta[2 * i]);
      parts[i].kind = kind;
      for (std::int64_t k = l.meta[2 * i + 1]; k < l.meta[2 * i + 3]; ++k) {
        const std::uint32_t c = l.cols[k];
        parts[i].neighbors.push_back(owner_ranges[c >> kOwnerShift].lb +
                                     (c & kOffsetMask));
      }
    }
    return parts;
  };
  auto lp = unpack(local, PartKind::local);
  auto rp = unpack(remote, PartKind::remote);
  // The implicit mapping, spelled out with the reference's own rules.
  auto warps = mapping == MappingMode::interleaved ? interleave(lp, rp, cfg.dist)
                                                   : map_segregated(lp, rp, cfg.dist);
  return map_to_blocks(std::move(lp), std::move(rp), std::move(warps), cfg, dim);
}

FlatPlan build_flat_plan(const CsrGraph& g, const WorkloadSplit& split,
                         const NePlacement& placement, std::uint32_t gpu,
                         const KernelConfig& cfg, std::uint64_t dim,
                         MappingMode mapping, Granularity granularity) {
  if (gpu >= split.num_gpus) throw InputError("split_local_remote: gpu_id out of range");
  if (split.num_nodes != g.num_nodes || placement.num_nodes != g.num_nodes)
    throw InputError("split_local_remote: inconsistent node counts");
  // Same check order as build_launch_plan: ps, dist, wpb.
  if (granularity == Granularity::partitioned) require_ps(cfg.ps);
  require_dist(cfg.dist);
  require_wpb(cfg.wpb);
  if (placement.num_gpus > kMaxOwners)
    throw ConfigError("flat plan: more than 16 embedding owners");
  for (const auto& r : placement.ranges)
    if (r.size() > kOffsetMask + 1ull)
      throw ConfigError("flat plan: shard exceeds 2^28 rows");

  FlatPlan fp;
  fp.gpu = gpu;
  const NodeRange chunk = split.chunk_ranges[gpu];
  fp.first_target = chunk.lb;
  fp.rows = chunk.size();
  fp.cfg = cfg;
  fp.dim = dim;
  fp.mapping = mapping;
  fp.granularity = granularity;
  fp.owner_ranges = placement.ranges;
  if (fp.rows > 0x7fffffffull) throw ConfigError("flat plan: chunk exceeds 2^31 rows");

  const OwnerIndex owner(placement);
  const std::uint32_t ps = cfg.ps;
  auto n_parts = [&](std::uint64_t n) -> std::uint64_t {
    if (n == 0) return 0;
    return granularity == Granularity::partitioned ? (n + ps - 1) / ps : 1;
  };

  // Pass 1: per slice of rows, count edges and partitions of each kind.
  const unsigned slices = std::max(1u, detail::host_threads() * 4);
  struct Tally {
    std::uint64_t le = 0, re = 0, lp = 0, rp = 0;
  };
  std::vector<Tally> tally(slices + 1);
  detail::parallel_slices(fp.rows, slices, [&](unsigned t, std::uint64_t b, std::uint64_t e) {
    Tally s;
    for (std::uint64_t r = b; r < e; ++r) {
      std::uint64_t nl = 0, nr = 0;
      for (NodeId nb : g.neighbors(chunk.lb + r)) (owner(nb) == gpu ? nl : nr)++;
      s.le += nl;
      s.re += nr;
      s.lp += n_parts(nl);
      s.rp += n_parts(nr);
    }
    tally[t + 1] = s;
  });
  for (unsigned t = 1; t <= slices; ++t) {  // inclusive scan -> slice offsets
    tally[t].le += tally[t - 1].le;
    tally[t].re += tally[t - 1].re;
    tally[t].lp += tally[t - 1].lp;
    tally[t].rp += tally[t - 1].rp;
  }
  const Tally tot = tally[slices];
  if (tot.le > 0x7fffffffull || tot.re > 0x7fffffffull)
    throw ConfigError("flat plan: more than 2^31 columns of one kind");
  fp.local.cols.resize(tot.le);
  fp.remote.cols.resize(tot.re);
  fp.local.meta.assign(2 * (tot.lp + 1), 0);
  fp.remote.meta.assign(2 * (tot.rp + 1), 0);
  fp.local.meta[2 * tot.lp] = -1;
  fp.local.meta[2 * tot.lp + 1] = static_cast<std::int32_t>(tot.le);
  fp.remote.meta[2 * tot.rp] = -1;
  fp.remote.meta[2 * tot.rp + 1] = static_cast<std::int32_t>(tot.re);

  // Pass 2: fill columns (order kept within each kind) and partition records.
  detail::parallel_slices(fp.rows, slices, [&](unsigned t, std::uint64_t b, std::uint64_t e) {
    std::uint64_t le = tally[t].le, re = tally[t].re, lp = tally[t].lp, rp = tally[t].rp;
    for (std::uint64_t r = b; r < e; ++r) {
      const std::uint64_t l0 = le, r0 = re;
      for (NodeId nb : g.neighbors(chunk.lb + r)) {
        const std::uint32_t o = owner(nb);
        const std::uint32_t packed =
            (o << kOwnerShift) | static_cast<std::uint32_t>(nb - placement.ranges[o].lb);
        if (o == gpu)
          fp.local.cols[le++] = packed;
        else
          fp.remote.cols[re++] = packed;
      }
      auto emit = [&](FlatPartList& l, std::uint64_t& pi, std::uint64_t c0,
                      std::uint64_t c1) {
        if (c1 == c0) return;
        const std::uint64_t step =
            granularity == Granularity::partitioned ? ps : (c1 - c0);
        for (std::uint64_t c = c0; c < c1; c += step, ++pi) {
          l.meta[2 * pi] = static_cast<std::int32_t>(r);
          l.meta[2 * pi + 1] = static_cast<std::int32_t>(c);
        }
      };
      emit(fp.local, lp, l0, le);
      emit(fp.remote, rp, r0, re);
    }
  });
  return fp;
}

}  // namespace mgg

namespace mgg {

double HaloPlan::dedup_ratio() const {
  return rows.empty() ? 0.0 : static_cast<double>(cols.size()) / static_cast<double>(rows.size());
}

HaloPlan build_halo_plan(const FlatPlan& plan) {
  HaloPlan h;
  const auto& rc = plan.remote.cols;
  h.cols.resize(rc.size());
  if (rc.empty()) return h;
  // Packed ids order as (owner, offset): mark + compact per owner shard.
  std::vector<std::uint64_t> base(plan.owner_ranges.size() + 1, 0);
  for (std::size_t o = 0; o < plan.owner_ranges.size(); ++o)
    base[o + 1] = base[o] + plan.owner_ranges[o].size();
  const std::uint64_t total = base.back();
  auto dense = [&](std::uint32_t c) { return base[c >> kOwnerShift] + (c & kOffsetMask); };
  std::vector<std::uint32_t> slot(total, 0);  // 1 + halo row, 0 = unused
  detail::parallel_for(rc.size(), 1 << 18, [&](std::uint64_t b, std::uint64_t e) {
    for (std::uint64_t i = b; i < e; ++i)
      std::atomic_ref<std::uint32_t>(slot[dense(rc[i])]).store(1, std::memory_order_relaxed);
  });
  std::uint32_t next = 0;
  for (std::size_t o = 0; o + 1 < base.size(); ++o)
    for (std::uint64_t d = base[o]; d < base[o + 1]; ++d)
      if (slot[d]) {
        slot[d] = ++next;
        h.rows.push_back(static_cast<std::uint32_t>(o << kOwnerShift) |
                         static_cast<std::uint32_t>(d - base[o]));
      }
  if (next > kOffsetMask + 1u) throw ConfigError("halo plan: more than 2^28 halo rows");
  detail::parallel_for(rc.size(), 1 << 18, [&](std::uint64_t b, std::uint64_t e) {
    for (std::uint64_t i = b; i < e; ++i) h.cols[i] = slot[dense(rc[i])] - 1;
  });
  return h;
}

}  // namespace mgg
