/* internal_abi.h -- entry points shared by the translation units of
 * libpbkv.so that are NOT part of the public C ABI (include/pbkv.h). */
#ifndef PBKV_INTERNAL_ABI_H_
#define PBKV_INTERNAL_ABI_H_

#include <stdint.h>

#include "../../../include/pbkv.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Which tracked host tree (TrackedCacheTree::uid, 0 = none) the context's
 * mirror holds, and the change-log position it has applied: pbkv_mirror_sync
 * (host_tree.cpp) reads and advances them; pbkv_mirror_full resets the uid. */
int pbkv_internal_mirror_tag(pbkv_ctx* ctx, uint64_t** uid, int64_t** pos);

/* Sets the thread-local message pbkv_last_error(NULL) returns. */
void pbkv_internal_set_error(const char* msg);

#ifdef __cplusplus
}
#endif

#endif /* PBKV_INTERNAL_ABI_H_ */
