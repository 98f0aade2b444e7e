"""B200-native KVTuner hot path (arXiv 2502.04420): layer-wise mixed-precision KV-cache
quantisation and the decode attention that reads it.  The compute lives in libkvt.so (sm_100a
CUDA, C ABI in include/kvt.h); this package is its thin Python binding."""
from .kvt import (ABI_VERSION, BUFFER_NAMES, ERROR_NAMES, MODE_KIVI, MODE_PER_CHANNEL_ASYM, MODE_PER_TOKEN_ASYM, Config, KvtError,
                  LayerCache, LayerSpec, cache_buffer_sizes, combine_partials, decode_attention,
                  append_decode_attention, decode_attention_partial, decode_attention_partial_push, decode_plan, decode_workspace_bytes, dbscan, layer_sensitivity, lib, load_config,
                  page_bytes, pareto_prune, prune_and_cluster, quantize_append, search_space_log10, validate_spec)

__all__ = ["ABI_VERSION", "BUFFER_NAMES", "ERROR_NAMES", "MODE_KIVI", "MODE_PER_CHANNEL_ASYM", "MODE_PER_TOKEN_ASYM", "Config", "KvtError",
           "LayerCache", "LayerSpec", "cache_buffer_sizes", "combine_partials", "decode_attention",
           "append_decode_attention", "decode_attention_partial", "decode_attention_partial_push", "decode_plan", "decode_workspace_bytes", "dbscan", "layer_sensitivity", "lib", "load_config",
           "page_bytes", "pareto_prune", "prune_and_cluster", "quantize_append", "search_space_log10", "validate_spec"]
