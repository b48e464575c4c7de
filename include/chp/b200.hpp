// chp/b200.hpp -- device options of the B200 drop-in that the reference API
// has no place for.  Not part of the reference interface: a caller that
// never includes this header gets the reference behaviour on one device
// (CHP_DEVICE, default 0).
#pragma once

#include <vector>

namespace chp::b200 {

// Devices reducer::reduce splits its input over, in this process (SURVEY.md
// 8(e); include/chp_b200.h chp_pipeline_host64_sharded): contiguous equal
// slices, one per device, the partial Ls merged by one element-wise MIN --
// ncclAllReduce when `nccl` (distinct devices), else one peer-memory kernel
// on the first device.  The result is the single-device result bit for bit.
// The default comes from CHP_DEVICES ("0,1,2,3"; CHP_COMBINE=peer selects
// the peer combine, CHP_COMBINE=fused the shards folding straight into the
// first device's L over peer memory), else {CHP_DEVICE or 0}.  Per host thread, like the
// drop-in's device context.
void use_devices(const std::vector<int>& devices, bool nccl = true);
std::vector<int> devices();

}  // namespace chp::b200
