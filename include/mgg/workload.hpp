// Neighbor-partition / warp-mapping metadata builder.
//
// Two views of the same metadata:
//
//  * The reference's value types and functions (R:proj/include/pipeshard/
//    workload.hpp:30-131): LocalRemoteSplit, NeighborPartition, WarpTask,
//    WarpWorkload, BlockAssignment, KernelLaunchPlan, split_local_remote,
//    partition_neighbors, interleave, map_segregated, map_to_blocks,
//    build_launch_plan, validate_plan, canonical JSON. Same semantics and
//    error behaviour, for drop-in callers and bit-exact parity tests.
//
//  * FlatPlan, the device form the sm_100a aggregation kernel consumes: per
//    kind a (target_row, begin) pair per partition plus one packed 32-bit
//    column per neighbor ((owner << 28) | offset-in-owner-shard). Warps and
//    blocks stay implicit — warp w owns partitions [w·dist, (w+1)·dist) of
//    each kind (interleaved) and a block is wpb consecutive warps — exactly
//    the reference's interleave/map_to_blocks (R:proj/src/workload.cpp:
//    103-172). build_flat_plan goes straight from the CSR to this form in
//    parallel; expand() rebuilds the reference KernelLaunchPlan from it and
//    is what the parity tests compare bit-for-bit.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "mgg/costmodel.hpp"
#include "mgg/graph.hpp"
#include "mgg/placement.hpp"

namespace mgg {

enum class PartKind : std::uint8_t { local, remote };

struct LocalRemoteSplit {
  std::uint32_t gpu_id = 0;
  NodeId first_target = 0;
  CsrGraph local_csr;   // rows = chunk targets, cols = global ids
  CsrGraph remote_csr;
};

struct NeighborPartition {
  NodeId target = 0;
  PartKind kind = PartKind::local;
  std::vector<NodeId> neighbors;  // 1..ps global ids
  std::uint64_t size() const { return neighbors.size(); }
};

struct WarpTask {
  PartKind kind;
  std::uint32_t index;
  friend bool operator==(const WarpTask&, const WarpTask&) = default;
};

struct WarpWorkload {
  std::uint32_t warp_id = 0;
  std::vector<WarpTask> tasks;  // local group first, then remote group
};

struct BlockAssignment {
  std::uint32_t first_warp = 0;
  std::uint32_t warp_count = 0;
};

struct KernelLaunchPlan {
  KernelConfig cfg;
  std::uint64_t dim = 1;
  std::vector<NeighborPartition> local_parts;
  std::vector<NeighborPartition> remote_parts;
  std::vector<WarpWorkload> warps;
  std::vector<BlockAssignment> blocks;
  std::uint64_t smem_bytes_per_block = 0;
};

enum class MappingMode : std::uint8_t { interleaved, segregated };
enum class Granularity : std::uint8_t { partitioned, whole_list };

LocalRemoteSplit split_local_remote(const CsrGraph& g, const WorkloadSplit& split,
                                    const NePlacement& placement,
                                    std::uint32_t gpu_id);
std::vector<NeighborPartition> partition_neighbors(const CsrGraph& csr,
                                                   NodeId first_target,
                                                   PartKind kind,
                                                   std::uint32_t ps);
std::vector<WarpWorkload> interleave(const std::vector<NeighborPartition>& local_parts,
                                     const std::vector<NeighborPartition>& remote_parts,
                                     std::uint32_t dist);
std::vector<WarpWorkload> map_segregated(
    const std::vector<NeighborPartition>& local_parts,
    const std::vector<NeighborPartition>& remote_parts, std::uint32_t dist);
KernelLaunchPlan map_to_blocks(std::vector<NeighborPartition> local_parts,
                               std::vector<NeighborPartition> remote_parts,
                               std::vector<WarpWorkload> warps,
                               const KernelConfig& cfg, std::uint64_t dim);
KernelLaunchPlan build_launch_plan(const LocalRemoteSplit& lr,
                                   const KernelConfig& cfg, std::uint64_t dim,
                                   MappingMode mapping = MappingMode::interleaved,
                                   Granularity granularity = Granularity::partitioned);
void validate_plan(const KernelLaunchPlan& plan);

/// Canonical JSON with the reference's keys (R:proj/src/workload.cpp:
/// 252-339); from_json re-derives blocks and re-validates.
std::string plan_to_json(const KernelLaunchPlan& plan);
KernelLaunchPlan plan_from_json(const std::string& text);

// ---------------------------------------------------------------------------
// Device form

inline constexpr std::uint32_t kOwnerShift = 28;
inline constexpr std::uint32_t kOffsetMask = (1u << kOwnerShift) - 1;
inline constexpr std::uint32_t kMaxOwners = 16;

struct FlatPartList {
  /// 2·(n+1) int32: (target_row, begin) per partition; entry n is the
  /// sentinel (-1, number of columns). Partition i covers cols[begin_i,
  /// begin_{i+1}) because partitions tile the kind's CSR in order.
  std::vector<std::int32_t> meta{-1, 0};
  std::vector<std::uint32_t> cols;  // (owner << 28) | offset
  std::uint64_t num_parts() const { return meta.size() / 2 - 1; }
};

struct FlatPlan {
  std::uint32_t gpu = 0;
  NodeId first_target = 0;
  std::uint64_t rows = 0;  // chunk size
  KernelConfig cfg;
  std::uint64_t dim = 1;
  MappingMode mapping = MappingMode::interleaved;
  Granularity granularity = Granularity::partitioned;
  std::vector<NodeRange> owner_ranges;  // NE placement ranges (for expand)
  FlatPartList local, remote;

  std::uint64_t num_local_warps() const {  // segregated: local-group warps
    return (local.num_parts() + cfg.dist - 1) / cfg.dist;
  }
  std::uint64_t num_warps() const;
  std::uint64_t num_blocks() const { return (num_warps() + cfg.wpb - 1) / cfg.wpb; }

  /// Rebuild the reference KernelLaunchPlan (bit-exact parity view).
  KernelLaunchPlan expand() const;
};

/// Deduplicated remote fetch plan of one gpu (a B200 addition; metadata of
/// the partitions is unchanged): the distinct remote rows its remote
/// partitions read, sorted by (owner, offset) so each peer shard is read in
/// address order, and the remote columns re-pointed at that compact halo.
/// One layer's remote traffic becomes unique_rows·D·4 bytes instead of
/// remote_edges·D·4 (Reddit-shaped, 8 GPUs: ~60x fewer NVLink bytes).
struct HaloPlan {
  std::vector<std::uint32_t> rows;       // packed (owner << 28) | offset
  std::vector<std::uint32_t> cols;       // remote column i -> halo row
  double dedup_ratio() const;            // remote columns per halo row
};
HaloPlan build_halo_plan(const FlatPlan& plan);

/// Split + partition + (implicit) warp/block mapping for one gpu, straight
/// from the CSR, multi-threaded. Same errors as build_launch_plan for bad
/// ps/dist/wpb; ConfigError if the packed encoding cannot address the
/// graph (> 16 owners, shard > 2^28 rows, > 2^31 columns per kind).
FlatPlan build_flat_plan(const CsrGraph& g, const WorkloadSplit& split,
                         const NePlacement& placement, std::uint32_t gpu,
                         const KernelConfig& cfg, std::uint64_t dim,
                         MappingMode mapping = MappingMode::interleaved,
                         Granularity granularity = Granularity::partitioned);

}  // namespace mgg
