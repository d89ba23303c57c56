"""ctypes signatures of every symbol declared in include/hybridcache.h.

tests/test_abi.py checks that this table and the header agree and that the
built library exports every symbol.
"""
import ctypes as C

i, l, d, u64, vp, cp = C.c_int, C.c_long, C.c_double, C.c_uint64, C.c_void_p, C.c_char_p
ip, lp, dp, u16p = C.POINTER(C.c_int), C.POINTER(C.c_long), C.POINTER(C.c_double), C.POINTER(C.c_uint16)
u64p, fp = C.POINTER(C.c_uint64), C.POINTER(C.c_float)
vpp, cpp = C.POINTER(C.c_void_p), C.POINTER(C.c_char_p)


class ModelConfigC(C.Structure):
    _fields_ = [("num_layers", C.c_int), ("hidden_dim", C.c_int), ("num_heads", C.c_int),
                ("ffn_dim", C.c_int), ("vocab_size", C.c_int), ("tokens_per_block", C.c_int),
                ("bytes_per_scalar", C.c_int)]


class EngineOptionsC(C.Structure):
    _fields_ = [("max_batch", C.c_int), ("max_seq", C.c_int), ("weights_on_device", C.c_int),
                ("kv_host_cap", C.c_long), ("kv_gpu_cap", C.c_long), ("act_host_cap", C.c_long),
                ("act_gpu_cap", C.c_long), ("kv_on_gpu", C.c_int), ("host_layers", C.c_int),
                ("mode", C.c_int), ("alloc_act_host", C.c_long), ("alloc_kv_host", C.c_long),
                ("scaled", C.c_int), ("max_prefill_tokens", C.c_int), ("device", C.c_int),
                ("weight_layers", C.c_int), ("recompute_ratio", C.c_double), ("arch", C.c_int),
                ("tp", C.c_void_p), ("weight_share", C.c_void_p)]


cfgp = C.POINTER(ModelConfigC)
optp = C.POINTER(EngineOptionsC)

SIGNATURES = {
    # library
    "hc_last_error": (cp, []),
    "hc_abi_version": (i, []),
    "hc_device_count": (i, []),
    "hc_device_pci_bus_id": (i, [i, C.c_char_p, i]),
    "hc_set_device": (i, [i]),
    # model
    "hc_model_validate": (i, [cfgp]),
    "hc_model_preset": (i, [cp, cfgp]),
    "hc_generate_weights": (i, [cfgp, u64, i, i, u16p, u16p, u16p]),
    # cache
    "hc_cache_create": (i, [i, l, l, l, l, i, vpp]),
    "hc_cache_destroy": (i, [vp]),
    "hc_cache_create_request": (i, [vp, cp, i]),
    "hc_cache_append_block": (i, [vp, cp, i, ip, ip]),
    "hc_cache_fill_token": (i, [vp, cp]),
    "hc_cache_free_request": (i, [vp, cp]),
    "hc_cache_context_len": (i, [vp, cp, ip]),
    "hc_cache_blocks_by_kind": (i, [vp, cp, lp, lp]),
    "hc_cache_free_blocks": (i, [vp, i, i, lp]),
    "hc_cache_capacity": (i, [vp, i, i, lp]),
    "hc_cache_table": (i, [vp, cp, ip, ip, ip, ip, i, ip]),
    "hc_cache_dump_json": (i, [vp, cp, l, lp]),
    "hc_bytes_of": (i, [i, i, i, i, u64p]),
    # planner
    "hc_next_block_kind": (i, [l, l, l, l, ip]),
    "hc_fit_linear": (i, [dp, dp, i, dp]),
    "hc_initial_cache_allocation": (i, [dp, i, l, lp]),
    "hc_alloc_remaining": (i, [dp, dp, i, l, l, lp]),
    "hc_plan_host_allocation": (i, [dp, dp, i, l, lp]),
    "hc_plan_hbm_residency": (i, [cfgp, l, l, d, dp, lp]),
    "hc_plan_hbm_tiers": (i, [cfgp, l, l, d, d, dp, i, dp, lp, dp]),
    "hc_planned_times": (i, [dp, i, l, l, l, dp]),
    "hc_plan_host_min_step": (i, [cfgp, l, l, d, dp, dp, lp, dp]),
    "hc_bundle_from_samples": (i, [dp, dp, i, dp, dp, i, d, cfgp, dp]),
    "hc_budget_for": (i, [d, cfgp, d, dp]),
    "hc_flop_count": (i, [i, cfgp, l, i, dp]),
    "hc_weight_bytes": (i, [cfgp, u64p]),
    # mini-batch packer
    "hc_form_minibatches": (i, [i, cpp, lp, lp, l, l, dp, i, ip, ip, ip]),
    "hc_brute_force_pack": (i, [i, cpp, lp, lp, l, l, dp, i, ip, ip, ip]),
    "hc_cost_fb": (i, [l, l, dp, i, dp]),
    "hc_default_packer": (i, [d, cfgp, lp]),
    # engine
    "hc_engine_create": (i, [cfgp, u64, i, i, optp, vpp]),
    "hc_engine_create_from_f64": (i, [cfgp, i, dp, dp, C.POINTER(dp), optp, vpp]),
    "hc_tp_nccl_unique_id": (i, [C.c_char_p]),
    "hc_tp_create_nccl": (i, [C.c_char_p, C.c_char_p, i, i, i, vpp]),
    "hc_tp_create_local_group": (i, [i, vpp]),
    "hc_tp_local_member": (i, [vp, i, vpp]),
    "hc_tp_create_emulated": (i, [i, i, vpp]),
    "hc_tp_destroy": (i, [vp, i]),
    "hc_engine_create_from_f64_opt": (i, [cfgp, i, dp, dp, C.POINTER(dp), C.POINTER(dp), dp, optp, vpp]),
    "hc_engine_destroy": (i, [vp]),
    "hc_engine_prefill": (i, [vp, i, cpp, ip, ip]),
    "hc_engine_admit_synthetic": (i, [vp, i, cpp, ip, u64]),
    "hc_engine_fill_pools": (i, [vp, u64]),
    "hc_engine_set_minibatching": (i, [vp, l, l, dp]),
    "hc_engine_set_fused_recompute": (i, [vp, i, ip]),
    "hc_engine_advance_synthetic": (i, [vp, i, cpp, i]),
    "hc_engine_decode_step": (i, [vp, i, cpp, ip, u16p, fp, ip]),
    "hc_engine_free_request": (i, [vp, cp]),
    "hc_engine_configure_cache": (i, [vp, l, l, l, l, i, i, l, l, i, d]),
    "hc_engine_forward_trace": (i, [vp, ip, i, u16p, u16p, u16p, u16p]),
    "hc_engine_layer_forward": (i, [vp, i, u16p, i, u16p, u16p, u16p]),
    "hc_engine_cache": (i, [vp, vpp]),
    "hc_engine_read_block": (i, [vp, i, i, i, i, u16p]),
    "hc_engine_read_weights": (i, [vp, i, u16p]),
    "hc_engine_capture_inputs": (i, [vp, i]),
    "hc_engine_captured_inputs": (i, [vp, u16p, l]),
    "hc_engine_last_stats": (i, [vp, dp]),
    "hc_engine_set_profile": (i, [vp, i]),
    "hc_engine_set_graphs": (i, [vp, i]),
    "hc_engine_trace_json": (i, [vp, cp, l, lp]),
    "hc_engine_time_kv_gen": (i, [vp, i, i, dp]),
    "hc_engine_time_load_kv": (i, [vp, i, i, dp]),
    # kernels (host buffers in / out)
    "hc_gemm_f16": (i, [i, i, i, i, u16p, u16p, vp, i]),
    "hc_gemm_f16_splitk": (i, [i, i, i, i, u16p, u16p, u16p, i, i]),
    "hc_gemm_f16_wstream": (i, [i, i, i, i, u16p, u16p, u16p, u16p, vp, i]),
    "hc_gemm_bench": (i, [i, i, i, i, i, i, dp]),
    "hc_recompute_kv_paged": (i, [i, i, i, i, u16p, u16p, ip, i, u16p, i]),
    "hc_decode_attention": (i, [i, i, i, i, u16p, u16p, l, u16p, l, ip, i, ip, ip, i, i, u16p]),
    "hc_prefill_attention": (i, [i, i, i, i, u16p, i, u16p]),
}
