// ORACLE SHIM (test infrastructure only): the image ships only the single-header
// nlohmann/json 3.11.3 (inside cudnn_frontend), not json_fwd.hpp; the full header
// declares everything json_fwd.hpp would. oracle/Makefile adds its directory.
#pragma once
#include <nlohmann/json.hpp>
