// refine.cu — A9/A10 placeholder (filled in with the refinement rows).
#include "internal.cuh"

namespace nrt {
nrt_status refine(nrt_scene, nrt_paths, const nrt_refine_desc*, nrt_paths, cudaStream_t) {
    return set_error(NRT_E_STATE, "refinement not built yet");
}
}  // namespace nrt
