// ORACLE / TEST INFRASTRUCTURE ONLY.
// config.cpp needs nlohmann/json (absent here), but metrics.cpp only uses its
// EstimatorKind name mapping (config.cpp:223-230), restated here so the reference's own
// rmse_sweep (metrics.cpp:92-120) links into oracle/_ref/libofdmref.so.
#include <string>

#include "ofdmradar/config.hpp"

namespace ofdmradar {

std::string to_string(EstimatorKind k) {
    switch (k) {
        case EstimatorKind::Ls: return "ls";
        case EstimatorKind::DftCe: return "dft-ce";
        case EstimatorKind::ZcpLs: return "zcp-ls";
    }
    return "?";
}

}  // namespace ofdmradar
