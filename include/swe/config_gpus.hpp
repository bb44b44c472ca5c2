// swe/config_gpus.hpp -- backend.gpus in the run configuration (SURVEY.md
// §8(f) row 4; reference io.hpp:361-374 parses the "backend" object and
// rejects unknown keys).  Kept separate from the reference's parser, which
// compiles and behaves unchanged: the B200 keys are taken out of the config
// text first and applied to the BackendSpec the parser returns.
//
//   BackendSpec ext;
//   const std::string rest = swe::split_backend_gpus(text, ext);
//   Config c = parse_config(rest);                  // the reference's parser
//   swe::apply_backend_gpus(ext, c.backend);
//
// Keys: "gpus" (int >= 1), "devices" (array of CUDA ordinals, one per GPU
// part), "device" (first ordinal when "devices" is absent).  Needs
// nlohmann/json (json.hpp), as the reference's io.hpp does.
#pragma once

#include <string>
#include <vector>

#include <json.hpp>

#include "swe/core.hpp"
#include "swe/engine.hpp"

namespace swe {

inline std::string split_backend_gpus(const std::string& json_text, BackendSpec& ext) {
  nlohmann::json j;
  try {
    j = nlohmann::json::parse(json_text);
  } catch (const nlohmann::json::parse_error& e) {
    throw config_error(std::string("config is not valid JSON: ") + e.what());
  }
  if (!j.is_object() || !j.contains("backend") || !j.at("backend").is_object()) return json_text;
  auto& jb = j.at("backend");
  try {
    if (jb.contains("gpus")) {
      ext.gpus = jb.at("gpus").get<int>();
      if (ext.gpus < 1) throw config_error("backend.gpus must be >= 1");
      jb.erase("gpus");
    }
    if (jb.contains("device")) {
      ext.device = jb.at("device").get<int>();
      jb.erase("device");
    }
    if (jb.contains("devices")) {
      ext.devices = jb.at("devices").get<std::vector<int>>();
      if (!ext.devices.empty() && static_cast<int>(ext.devices.size()) != ext.gpus)
        throw config_error("backend.devices must list backend.gpus devices");
      jb.erase("devices");
    }
  } catch (const nlohmann::json::exception& e) {
    throw config_error(std::string("config: backend: ") + e.what());
  }
  return j.dump();
}

inline void apply_backend_gpus(const BackendSpec& ext, BackendSpec& b) {
  b.gpus = ext.gpus;
  b.device = ext.device;
  b.devices = ext.devices;
}

}  // namespace swe
