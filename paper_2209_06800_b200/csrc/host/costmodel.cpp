// Analytical model and hardware profiles (see include/mgg/costmodel.hpp).
#include "mgg/costmodel.hpp"

#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <sstream>

#include <nlohmann/json.hpp>

#include "mgg/errors.hpp"

namespace mgg {

std::uint64_t wpw(const KernelConfig& c, std::uint64_t dim) {
  return 2ull * c.ps * dim * c.dist;
}

std::uint64_t smem(const KernelConfig& c, std::uint64_t dim) {
  // neighbor ids (int) + partial results and fetched rows (float), 4 B each
  return 4ull * c.ps * c.wpb + 8ull * c.wpb * dim;
}

std::uint64_t launch_smem(const KernelConfig&, std::uint64_t) {
  return 16 * sizeof(void*);
}

LaunchGeometry launch_geometry(std::uint64_t n_local_parts,
                               std::uint64_t n_remote_parts,
                               const KernelConfig& c,
                               const HardwareProfile& hw) {
  LaunchGeometry g;
  const std::uint64_t longest = n_local_parts > n_remote_parts ? n_local_parts
                                                                : n_remote_parts;
  g.num_warps = (longest + c.dist - 1) / c.dist;
  g.num_blocks = (g.num_warps + c.wpb - 1) / c.wpb;
  g.blocks_per_sm =
      static_cast<double>(g.num_blocks) / static_cast<double>(hw.num_sms);
  return g;
}

namespace {
std::string range_msg(const char* name, std::uint32_t v, std::uint32_t hi) {
  return std::string(name) + "=" + std::to_string(v) + " outside [1," +
         std::to_string(hi) + "]";
}
}  // namespace

std::vector<Violation> validate(const KernelConfig& c,
                                const HardwareProfile& hw, std::uint64_t dim) {
  std::vector<Violation> out;
  if (c.ps < 1 || c.ps > kMaxPs)
    out.push_back({"ps range", range_msg("ps", c.ps, kMaxPs)});
  if (c.dist < 1 || c.dist > kMaxDist)
    out.push_back({"dist range", range_msg("dist", c.dist, kMaxDist)});
  if (c.wpb < 1 || c.wpb > kMaxWpb)
    out.push_back({"wpb range", range_msg("wpb", c.wpb, kMaxWpb)});
  if (c.wpb > hw.max_warps_per_sm)
    out.push_back({"wpb capacity", "wpb=" + std::to_string(c.wpb) +
                                       " exceeds " +
                                       std::to_string(hw.max_warps_per_sm) +
                                       " warp slots"});
  if (c.ps >= 1 && c.wpb >= 1 && smem(c, dim) > hw.smem_per_sm_bytes)
    out.push_back({"smem", std::to_string(smem(c, dim)) +
                               " bytes per block > " +
                               std::to_string(hw.smem_per_sm_bytes) +
                               " bytes per SM"});
  return out;
}

HardwareProfile builtin_profile(const std::string& name) {
  HardwareProfile hw;  // defaults are the a100 preset
  if (name == "a100") return hw;
  if (name == "v100") {
    hw.name = "v100";
    hw.num_sms = 80;
    hw.smem_per_sm_bytes = 96 * 1024;
    hw.device_mem_bytes = 16ull << 30;
    return hw;
  }
  if (name == "desk") {
    hw.name = "desk";
    hw.num_sms = 8;
    hw.max_warps_per_sm = 2;
    hw.smem_per_sm_bytes = 96 * 1024;
    hw.device_mem_bytes = 1ull << 30;
    return hw;
  }
  if (name == "b200") {
    // cudaGetDeviceProperties on the pool's B200s: 148 SMs, 64 warps/SM,
    // 228 KB smem/SM, 183,359 MiB HBM3e. Latencies in SM cycles at the
    // 1965 MHz max clock: local = K5 chase probe (417.6 ns HBM dependent
    // load), remote = NVLink 5 peer load ~1.86 us; per-element costs are
    // sub-cycle on B200 and clamp to the schema's integer minimum.
    hw.name = "b200";
    hw.num_sms = 148;
    hw.max_warps_per_sm = 64;
    hw.smem_per_sm_bytes = 228 * 1024;
    hw.device_mem_bytes = 183359ull << 20;
    hw.page_bytes = 4096;
    hw.barrier_cycles = 4000;
    hw.lat = {3650, 820, 1, 1, 1};  // profiles/b200.json "source"
    return hw;
  }
  throw ConfigError("unknown hardware profile '" + name + "'");
}

namespace {

HardwareProfile from_json_obj(const nlohmann::json& j) {
  HardwareProfile hw;
  j.at("name").get_to(hw.name);
  j.at("numSMs").get_to(hw.num_sms);
  j.at("maxWarpsPerSM").get_to(hw.max_warps_per_sm);
  j.at("smemPerSMBytes").get_to(hw.smem_per_sm_bytes);
  j.at("deviceMemBytes").get_to(hw.device_mem_bytes);
  if (j.contains("pageBytes")) j.at("pageBytes").get_to(hw.page_bytes);
  if (j.contains("barrierCycles")) j.at("barrierCycles").get_to(hw.barrier_cycles);
  if (j.contains("latencies")) {
    const auto& l = j.at("latencies");
    l.at("remoteGetBase").get_to(hw.lat.remote_get_base);
    l.at("localLoadBase").get_to(hw.lat.local_load_base);
    l.at("perElemRemote").get_to(hw.lat.per_elem_remote);
    l.at("perElemLocal").get_to(hw.lat.per_elem_local);
    l.at("perElemCompute").get_to(hw.lat.per_elem_compute);
  }
  if (hw.num_sms < 1 || hw.max_warps_per_sm < 1)
    throw ParseError("profile: counts must be >= 1", 0);
  return hw;
}

}  // namespace

std::string profile_to_json(const HardwareProfile& hw) {
  nlohmann::json j{{"name", hw.name},
                   {"numSMs", hw.num_sms},
                   {"maxWarpsPerSM", hw.max_warps_per_sm},
                   {"smemPerSMBytes", hw.smem_per_sm_bytes},
                   {"deviceMemBytes", hw.device_mem_bytes},
                   {"pageBytes", hw.page_bytes},
                   {"barrierCycles", hw.barrier_cycles},
                   {"latencies",
                    {{"remoteGetBase", hw.lat.remote_get_base},
                     {"localLoadBase", hw.lat.local_load_base},
                     {"perElemRemote", hw.lat.per_elem_remote},
                     {"perElemLocal", hw.lat.per_elem_local},
                     {"perElemCompute", hw.lat.per_elem_compute}}}};
  return j.dump(2);
}

HardwareProfile profile_from_json(const std::string& text) {
  try {
    return from_json_obj(nlohmann::json::parse(text));
  } catch (const nlohmann::json::exception& e) {
    throw ParseError(std::string("profile: ") + e.what(), 0);
  }
}

HardwareProfile load_profile(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw InputError("cannot open profile file '" + path + "'");
  std::stringstream ss;
  ss << in.rdbuf();
  try {
    return from_json_obj(nlohmann::json::parse(ss.str()));
  } catch (const nlohmann::json::exception& e) {
    throw ParseError("profile '" + path + "': " + e.what(), 0);
  }
}

HardwareProfile resolve_profile(const std::string& name_or_path,
                                const std::string& profile_dir) {
  namespace fs = std::filesystem;
  std::error_code ec;
  if (fs::is_regular_file(name_or_path, ec)) return load_profile(name_or_path);
  std::string dir = profile_dir;
  if (dir.empty())
    if (const char* env = std::getenv("PIPESHARD_PROFILE_DIR")) dir = env;
  if (!dir.empty()) {
    const fs::path f = fs::path(dir) / (name_or_path + ".json");
    if (fs::exists(f, ec)) return load_profile(f.string());
  }
  return builtin_profile(name_or_path);
}

std::uint64_t remote_partition_bytes(std::uint64_t part_size, std::uint64_t dim,
                                     Transport transport,
                                     std::uint64_t page_bytes) {
  const std::uint64_t row = dim * 4;
  if (transport == Transport::fine_grained) return part_size * row;
  return part_size * ((row + page_bytes - 1) / page_bytes) * page_bytes;
}

}  // namespace mgg
