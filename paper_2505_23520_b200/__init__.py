"""B200-native AnchorAttention prefill stack (arXiv 2505.23520).

* ``paper_2505_23520_b200.anchorattn`` — pybind11 module with the reference's
  Python names (``BlockConfig``, ``HeadWorkload``, ``anchor_attention``,
  ``identify_stripes`` ...) over the C++ ``anchorattn::`` shim.
* ``paper_2505_23520_b200.capi`` — ctypes binding of the C ABI
  (include/anchorattn_capi.h) for device-resident, multi-head/GQA tensors.
* ``paper_2505_23520_b200.workloads`` — O(N*d) synthetic sink/stripe heads.
* ``paper_2505_23520_b200.sharding`` — KV-head sharding across ranks.
"""
__all__ = ["capi", "workloads", "build"]
