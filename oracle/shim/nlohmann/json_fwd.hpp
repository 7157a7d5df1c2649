// Test-infrastructure shim (oracle only): the reference's pipeline.hpp includes
// <nlohmann/json_fwd.hpp> from its un-shipped vendor/ tree. The container has
// nlohmann/json v3.11.3 (cudnn_frontend thirdparty); forward to the full header.
#pragma once
#include <nlohmann/json.hpp>
