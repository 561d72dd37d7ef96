"""ctypes binding of libslimsell_b200.so (include/slimsell_b200.h).

The shared library is the product: there is no CPU fallback. Importing this
module without the built library raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SSB_LIB", os.path.join(HERE, "libslimsell_b200.so"))  # override: experiments
CSRC = os.path.join(HERE, "csrc")

SSB_OK, SSB_EINVAL, SSB_ERANGE, SSB_ECAP, SSB_ECUDA, SSB_ENOMEM, SSB_EPARSE = range(7)

i64p = C.POINTER(C.c_int64)
i32p = C.POINTER(C.c_int32)


class LayoutInfo(C.Structure):
    _fields_ = [(k, C.c_int64) for k in ("C", "sigma", "n", "n_padded", "n_chunks", "nonzeros",
                                         "n_cells", "padding", "max_chunk_len", "range_begin",
                                         "range_end", "range_cells", "range_segments")]


class BfsOptionsC(C.Structure):
    _fields_ = [("variant", C.c_int32), ("slimwork", C.c_int32), ("slimchunk_len", C.c_int64),
                ("schedule", C.c_int32), ("workers", C.c_int32), ("max_iterations", C.c_int64),
                ("want_parents", C.c_int32), ("selmax_compat", C.c_int32)]


class IterStatsC(C.Structure):
    _fields_ = [(k, C.c_int64) for k in ("iteration", "elapsed_ns", "chunks_processed",
                                         "chunks_skipped", "subchunks_processed",
                                         "columns_processed", "frontier_size")]


def build(verbose: bool = False, force: bool = False) -> str:
    """Compile libslimsell_b200.so for sm_100a (nvcc; no GPU needed).
    force=True recompiles every source (make -B)."""
    cmd = ["make", "-s", "-C", CSRC, f"-j{min(8, os.cpu_count() or 1)}"] + (["-B"] if force else [])
    out = subprocess.run(cmd, capture_output=not verbose, text=True)
    if out.returncode != 0:
        raise RuntimeError(f"building libslimsell_b200.so failed:\n{out.stdout}\n{out.stderr}")
    return LIB_PATH


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing; run paper_2010_09913_b200._lib.build() "
                          "(or __graft_entry__.build()) first — there is no CPU fallback")
    L = C.CDLL(LIB_PATH)
    vp = C.c_void_p
    pvp = C.POINTER(vp)
    sig = {
        "ssb_last_error": (C.c_char_p, []),
        "ssb_abi_version": (C.c_int, []),
        "ssb_set_device": (C.c_int, [C.c_int]),
        "ssb_edges_from_pairs": (C.c_int, [i64p, C.c_int64, C.c_int64, pvp]),
        "ssb_gen_kronecker": (C.c_int, [C.c_int64, C.c_int64, C.c_uint64, C.POINTER(C.c_double), pvp]),
        "ssb_gen_erdos_renyi": (C.c_int, [C.c_int64, C.c_double, C.c_uint64, pvp]),
        "ssb_edges_from_edge_list": (C.c_int, [C.c_char_p, C.c_int64, C.c_int, pvp]),
        "ssb_edges_from_matrix_market": (C.c_int, [C.c_char_p, C.c_int64, pvp]),
        "ssb_parse_edge_list": (C.c_int, [C.c_char_p, C.c_int64, C.c_int, C.POINTER(i64p), i64p, i64p]),
        "ssb_parse_matrix_market": (C.c_int, [C.c_char_p, C.c_int64, C.POINTER(i64p), i64p, i64p]),
        "ssb_free": (None, [vp]),
        "ssb_edges_info": (C.c_int, [vp, i64p, i64p]),
        "ssb_edges_export": (C.c_int, [vp, i64p]),
        "ssb_to_csr": (C.c_int, [vp, i64p, i64p]),
        "ssb_edges_destroy": (None, [vp]),
        "ssb_build_slimsell": (C.c_int, [vp, C.c_int64, C.c_int64, pvp]),
        "ssb_build_slimsell_range": (C.c_int, [vp, C.c_int64, C.c_int64, C.c_int64, C.c_int64, pvp]),
        "ssb_build_slimsell_segments": (C.c_int, [vp, C.c_int64, C.c_int64, i64p, C.c_int64, pvp]),
        "ssb_graph_from_layout": (C.c_int, [C.c_int64, C.c_int64, C.c_int64, C.c_int64, i64p, C.c_int64,
                                            i64p, i64p, C.c_int64, i64p, pvp]),
        "ssb_graph_info": (C.c_int, [vp, C.POINTER(LayoutInfo)]),
        "ssb_graph_export": (C.c_int, [vp, i64p, i64p, i64p, i64p, i64p]),
        "ssb_graph_export_col32": (C.c_int, [vp, i32p]),
        "ssb_graph_degrees": (C.c_int, [vp, i64p]),
        "ssb_bfs_last_timing": (C.c_int, [vp, C.POINTER(C.c_double), i64p]),
        "ssb_graph_destroy": (None, [vp]),
        "ssb_spmv_step": (C.c_int, [vp, C.c_int, i64p, i64p, C.c_int64, C.c_int64]),
        "ssb_spmv_step_device": (C.c_int, [vp, C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64,
                                           C.POINTER(C.c_double)]),
        "ssb_spmv_segment": (C.c_int, [vp, C.c_int, i64p, i64p, C.c_int64, C.c_int64, C.c_int64]),
        "ssb_bfs_spmv": (C.c_int, [vp, C.c_int64, C.POINTER(BfsOptionsC), i64p, i64p, i64p,
                                   C.POINTER(IterStatsC), C.c_int64, i64p]),
        "ssb_bfs_spmv_batch": (C.c_int, [vp, i64p, C.c_int64, C.POINTER(BfsOptionsC), C.POINTER(i64p),
                                         C.POINTER(i64p), i64p, i64p]),
        "ssb_bfs_run": (C.c_int, [vp, C.c_int64, C.POINTER(BfsOptionsC), C.POINTER(IterStatsC),
                                  C.c_int64, i64p, C.POINTER(C.c_double)]),
        "ssb_bfs_fetch": (C.c_int, [vp, C.c_int, i64p, i64p, i64p]),
        "ssb_bfs_edges_traversed": (C.c_int, [vp, i64p]),
        "ssb_bfs_columns_swept": (C.c_int, [vp, i64p]),
        "ssb_bfs_traditional": (C.c_int, [vp, C.c_int64, i64p, i64p, C.POINTER(IterStatsC), C.c_int64, i64p]),
        "ssb_validate_bfs": (C.c_int, [vp, C.c_int64, i64p, i64p, C.c_int, i64p, C.c_char_p, C.c_int64]),
        "ssb_validate_bfs_exact": (C.c_int, [vp, vp, C.c_int64, i64p, i64p, C.c_int, i64p, C.c_char_p,
                                             C.c_int64]),
        "ssb_bfs_shard_begin": (C.c_int, [vp, C.c_int64, C.POINTER(BfsOptionsC), C.c_int64, C.c_int64]),
        "ssb_bfs_shard_step": (C.c_int, [vp, C.POINTER(IterStatsC), C.c_void_p]),
        "ssb_bfs_shard_exchange": (C.c_int, [vp, C.c_void_p, C.c_int64]),
        "ssb_bfs_shard_fetch": (C.c_int, [vp, C.c_int, i64p, i64p]),
        "ssb_graph_stream": (C.c_int, [vp, C.POINTER(C.c_void_p)]),
        "ssb_ctx_create": (C.c_int, [C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_void_p)]),
        "ssb_partition_segments": (C.c_int, [i32p, C.c_int64, C.c_int64, C.c_int, C.c_int, i64p]),
        "ssb_ctx_destroy": (None, [vp]),
        "ssb_ctx_build": (C.c_int, [vp, vp, C.c_int64, C.c_int64, C.c_int, C.POINTER(C.c_void_p)]),
        "ssb_sharded_info": (C.c_int, [vp, C.POINTER(C.c_int), i64p, i64p, i64p]),
        "ssb_sharded_bfs": (C.c_int, [vp, C.c_int64, C.POINTER(BfsOptionsC), i64p, i64p, i64p,
                                      C.POINTER(IterStatsC), C.c_int64, i64p, C.POINTER(C.c_double)]),
        "ssb_sharded_destroy": (None, [vp]),
        "ssb_bfs_shard_begin_async": (C.c_int, [vp, C.c_int64, C.POINTER(BfsOptionsC), C.c_int64, C.c_int64]),
        "ssb_bfs_shard_step_async": (C.c_int, [vp, C.c_void_p]),
        "ssb_bfs_shard_exchange_async": (C.c_int, [vp, C.c_void_p]),
        "ssb_bfs_shard_front": (C.c_int, [vp, C.c_int64, i64p]),
        "ssb_bfs_shard_finish": (C.c_int, [vp, C.c_int64, C.POINTER(IterStatsC), C.c_int64,
                                           C.POINTER(C.c_double)]),
        "ssb_p2p_window": (C.c_int, [vp, C.c_void_p, i64p]),
        "ssb_p2p_attach": (C.c_int, [vp, C.c_int, C.c_int, C.c_void_p, C.c_int64, C.c_int64]),
        "ssb_bfs_p2p": (C.c_int, [vp, C.c_int64, C.POINTER(BfsOptionsC), C.POINTER(IterStatsC), C.c_int64,
                                  i64p, C.POINTER(C.c_double)]),
        "ssb_p2p_attach_segments": (C.c_int, [vp, C.c_int, C.c_int, C.c_void_p, i64p, C.c_int64]),
        "ssb_bfs_p2p_group": (C.c_int, [pvp, C.c_int, i64p, i64p, C.c_int64, C.POINTER(BfsOptionsC),
                                        C.POINTER(IterStatsC), C.c_int64, i64p, C.POINTER(C.c_double)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


EXPORTED_SYMBOLS = None  # filled lazily by exported_symbols()


def header_symbols() -> list[str]:
    """Function names declared in include/slimsell_b200.h."""
    import re
    hdr = os.path.join(os.path.dirname(HERE), "include", "slimsell_b200.h")
    text = open(hdr).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(ssb_[a-z_0-9]+)\s*\(", text, re.M)))
