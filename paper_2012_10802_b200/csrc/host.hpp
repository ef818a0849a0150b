// host.hpp — host-side declarations shared by the extern "C" layer.
#pragma once

#include <string>

#include "common.cuh"

namespace rpdg {

void config_default(rpd_config* c);
void config_validate(const rpd_config& c);
void config_set(rpd_config* c, const std::string& key, const std::string& value);

}  // namespace rpdg
