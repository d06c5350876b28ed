// The analytical half of the runtime: Eq. 1-3 of the paper (R:PAPER.md:
// 427-453), the search-space constraints (R:PAPER.md:462-469) and the
// hardware profiles. Same names, formulas, ranges, JSON schema and profile
// resolution order as the reference (R:proj/include/pipeshard/
// costmodel.hpp:32-108, R:proj/src/costmodel.cpp:27-181), plus a measured
// `b200` preset and the smem the B200 aggregation kernel actually launches
// with (launch_smem), which differs from the paper's SMEM formula.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace mgg {

/// Per-operation cost model. In the reference these are abstract DES cycle
/// costs (R:proj/include/pipeshard/costmodel.hpp:32-38); the b200 preset
/// carries values re-fitted from measured B200 latencies (ns-scaled cycles).
struct LatencyModel {
  std::uint64_t remote_get_base = 384;
  std::uint64_t local_load_base = 128;
  std::uint64_t per_elem_remote = 1;
  std::uint64_t per_elem_local = 1;
  std::uint64_t per_elem_compute = 1;
};

struct HardwareProfile {
  std::string name = "a100";
  std::uint32_t num_sms = 108;
  std::uint32_t max_warps_per_sm = 64;
  std::uint64_t smem_per_sm_bytes = 164 * 1024;
  std::uint64_t device_mem_bytes = 40ull << 30;
  std::uint64_t page_bytes = 4096;
  std::uint64_t barrier_cycles = 64;
  LatencyModel lat;
};

/// (ps, dist, wpb); legal ranges ps∈[1,32], dist∈[1,16], wpb∈[1,16].
struct KernelConfig {
  std::uint32_t ps = 1;
  std::uint32_t dist = 1;
  std::uint32_t wpb = 1;
  friend bool operator==(const KernelConfig&, const KernelConfig&) = default;
};

struct LaunchGeometry {
  std::uint64_t num_warps = 0;
  std::uint64_t num_blocks = 0;
  double blocks_per_sm = 0.0;
};

struct Violation {
  std::string constraint;  // "ps range" | "dist range" | "wpb range" |
                           // "wpb capacity" | "smem"
  std::string detail;
};

inline constexpr std::uint32_t kMaxPs = 32;
inline constexpr std::uint32_t kMaxDist = 16;
inline constexpr std::uint32_t kMaxWpb = 16;

/// WPW = 2·ps·D·dist (Eq. 1).
std::uint64_t wpw(const KernelConfig& cfg, std::uint64_t dim);
/// SMEM = ps·wpb·4 + 2·wpb·D·4 (Eq. 1); the paper's layout, kept for
/// validate() parity with the reference.
std::uint64_t smem(const KernelConfig& cfg, std::uint64_t dim);
/// Dynamic shared memory the sm_100a aggregation kernel launches with:
/// a per-block copy of the peer base-pointer table (16 × 8 B). Rows are
/// staged in registers, not in the paper's smem layout.
std::uint64_t launch_smem(const KernelConfig& cfg, std::uint64_t dim);

/// Eq. 2-3 with ceilings (R:proj/src/costmodel.cpp:38-49).
LaunchGeometry launch_geometry(std::uint64_t n_local_parts,
                               std::uint64_t n_remote_parts,
                               const KernelConfig& cfg,
                               const HardwareProfile& hw);

/// Empty when admissible (R:proj/src/costmodel.cpp:51-77).
std::vector<Violation> validate(const KernelConfig& cfg,
                                const HardwareProfile& hw, std::uint64_t dim);

/// "a100", "v100", "desk" (reference presets) and "b200" (this build).
HardwareProfile builtin_profile(const std::string& name);
HardwareProfile load_profile(const std::string& path);
/// Exact file, then <profile_dir or $PIPESHARD_PROFILE_DIR>/<name>.json, then
/// built-ins (R:proj/src/costmodel.cpp:118-133).
HardwareProfile resolve_profile(const std::string& name_or_path,
                                const std::string& profile_dir = "");

std::string profile_to_json(const HardwareProfile& hw);
HardwareProfile profile_from_json(const std::string& text);

/// Remote transfer granularity (R:proj/include/pipeshard/sim.hpp:21-22).
enum class Transport : std::uint8_t { fine_grained, paged };

/// Bytes one remote partition of part_size neighbors moves: fine = size·D·4,
/// paged = size·ceil(4D/page)·page (R:proj/src/sim.cpp:503-518).
std::uint64_t remote_partition_bytes(std::uint64_t part_size, std::uint64_t dim,
                                     Transport transport,
                                     std::uint64_t page_bytes);

}  // namespace mgg
