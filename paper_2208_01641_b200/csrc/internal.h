// internal.h -- symbols shared between the runtime's translation units (not exported).
#pragma once
#include <cstddef>
#include <cstdint>
#include "../../include/lic.h"

// real (unpadded) frame pixels H*W of a codec
size_t lic_internal_frame_pixels(const lic_codec* c);
// a second codec with the same weights / geometry / device (own buffers): decoder GPU1 on its own stream
lic_status lic_internal_clone(const lic_codec* c, lic_codec** out);
// kernels this codec has launched
uint64_t lic_internal_launches(const lic_codec* c);
int lic_internal_zero_copy(const lic_codec* c);   // kernels touch pinned host planes in place
