"""Build and load ``libflint_b200.so`` (the CUDA engine behind include/flint_b200.h).

The library is compiled in-tree for sm_100a only
(``-gencode arch=compute_100a,code=sm_100a``) and loaded with ctypes.  There
is no fallback: if the library is missing or no GPU is visible, every engine
entry point raises :class:`~paper_2604_17550_b200.errors.EngineError`.
"""

from __future__ import annotations

import ctypes as C
import os
import shutil
import subprocess
from pathlib import Path

from .errors import EngineError

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
BUILD = PKG / "_build"
LIB = BUILD / "libflint_b200.so"
SOURCES = [PKG / "csrc" / "engine.cu", PKG / "csrc" / "capi.cu"]
HEADERS = [ROOT / "include" / "flint_b200.h", PKG / "csrc" / "engine_internal.h"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-fmad=false",                 # no FMA contraction: bit-exact fp64 cost model
    "-Xcompiler", "-fPIC",
]
# engine.cu is compiled once per kernel-variant group (compute streams | 8 with messages,
# engine.cu FL_BASE) so the groups build in parallel
ENGINE_PARTS = (1, 2, 4, 9, 10, 12, 512, 520)


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (Path(cand).exists() or cand == "nvcc"):
            return cand
    return "nvcc"


def _compile(out: Path, defines=(), verbose: bool = False) -> str:
    """nvcc every translation unit to an object (in parallel), then link `out`."""
    tmp = out.parent / (out.name + ".objs")
    tmp.mkdir(parents=True, exist_ok=True)
    inc = ["-I", str(ROOT / "include"), "-I", str(PKG / "csrc")]
    dflags = [f"-D{d}" for d in defines]
    jobs = [(PKG / "csrc" / "engine.cu", tmp / f"engine_{b}.o", [f"-DFL_BASE={b}"]) for b in ENGINE_PARTS]
    jobs.append((PKG / "csrc" / "capi.cu", tmp / "capi.o", []))
    procs = []
    for src, obj, extra in jobs:
        cmd = [nvcc(), *NVCC_FLAGS, *os.environ.get("FLINT_NVCC_EXTRA", "").split(), *dflags, *extra, *inc,
               "-c", str(src), "-o", str(obj)]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        procs.append(subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True))
    err = ""
    failed = False
    for p in procs:
        _, e = p.communicate()
        err += e
        failed |= p.returncode != 0
    if failed:
        raise EngineError("nvcc failed:\n" + err[-4000:])
    link = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", *[str(o) for _, o, _ in jobs],
            "-o", str(out)]
    res = subprocess.run(link, capture_output=True, text=True)
    shutil.rmtree(tmp, ignore_errors=True)
    if res.returncode != 0:
        raise EngineError("nvcc link failed:\n" + res.stderr[-4000:])
    return err


def build_variant(out: Path, defines=(), verbose: bool = False) -> str:
    """Compile the engine with extra -D flags into `out` (A/B experiments)."""
    return _compile(out, defines, verbose)


def build(force: bool = False, verbose: bool = False) -> Path:
    BUILD.mkdir(exist_ok=True)
    newest = max(p.stat().st_mtime for p in SOURCES + HEADERS)
    if not force and LIB.exists() and LIB.stat().st_mtime >= newest:
        return LIB
    _compile(Path(str(LIB) + ".tmp"), verbose=verbose)
    os.replace(str(LIB) + ".tmp", LIB)
    return LIB


P64 = C.POINTER(C.c_int64)
P32 = C.POINTER(C.c_int32)
PU8 = C.POINTER(C.c_uint8)
PF64 = C.POINTER(C.c_double)


class GraphDesc(C.Structure):
    _fields_ = [
        ("n_ranks", C.c_int32), ("rank_struct", P32), ("rank_graph_pos", P32),
        ("n_structs", C.c_int32), ("s_node_off", P32), ("s_tens_off", P32), ("s_init_off", P32),
        ("s_init_alloc", P64), ("s_ncoll", P32),
        ("node_kind", PU8), ("node_flags", PU8), ("node_id", P64), ("node_dur", P64),
        ("node_flops", P64), ("node_alloc", P64), ("node_coll_ord", P32),
        ("pred_off", P32), ("pred_idx", P32), ("succ_off", P32), ("succ_idx", P32),
        ("free_off", P32), ("free_tens", P32), ("init_list", P32),
        ("tens_bytes", P64), ("tens_cons_off", P32), ("tens_cons", P32),
        ("n_inst", C.c_int32), ("inst_kind", PU8), ("inst_n", P32), ("inst_bytes", P64),
        ("inst_lead_id", P64), ("inst_init_key", P64), ("inst_mem_off", P64),
        ("inst_mem_rank", P32), ("inst_mem_node", P32),
        ("coll_stride", C.c_int32), ("rank_coll_inst", P32),
        ("rank_value", P64), ("n_msg", C.c_int32), ("msg_send_rank", P32), ("msg_send_node", P32),
        ("msg_recv_rank", P32), ("msg_recv_node", P32), ("msg_bytes", P64), ("msg_send_id", P64),
        ("p2p_stride", C.c_int32), ("rank_p2p_msg", P32),
    ]


class Points(C.Structure):
    _fields_ = [
        ("n_points", C.c_int32), ("algo", PU8), ("topo_kind", PU8), ("bw", PF64),
        ("latency", P64), ("rows", P32), ("cols", P32), ("peak_flops", PF64),
        ("efficiency", PF64), ("compute_streams", C.c_int32),
    ]


class Outputs(C.Structure):
    _fields_ = [("status", P32), ("rows", P64), ("rank_stats", P64),
                ("ev_start", P64), ("ev_end", P64), ("link_busy", P64), ("link_cap", C.c_int32),
                ("trace", P64), ("trace_len", P32), ("trace_cap", C.c_int32)]


class PointsRaw(C.Structure):
    """fl_points with untyped pointers (same layout as Points): filled from raw addresses on the
    per-call path, where building typed ctypes pointers costs more than the call itself."""
    _fields_ = [(n, C.c_void_p if t not in (C.c_int32,) else t) for n, t in Points._fields_]


class OutputsRaw(C.Structure):
    _fields_ = [(n, C.c_void_p if t not in (C.c_int32,) else t) for n, t in Outputs._fields_]


_lib = None


def _header_abi_version() -> int:
    for line in (ROOT / "include" / "flint_b200.h").read_text().splitlines():
        if line.startswith("#define FL_ABI_VERSION"):
            return int(line.split()[2])
    raise EngineError("include/flint_b200.h has no FL_ABI_VERSION")


def lib():
    """Load the engine, (re)building it first when the in-tree library is missing or older than
    its sources, and refuse a library whose ABI version differs from include/flint_b200.h."""
    global _lib
    if _lib is not None:
        return _lib
    override = os.environ.get("FLINT_B200_LIB")     # A/B builds of the same engine (scripts/ab.py)
    if override:
        _lib = _bind(C.CDLL(override))
        return _lib
    stale = LIB.exists() and all(p.exists() for p in SOURCES + HEADERS) and \
        LIB.stat().st_mtime < max(p.stat().st_mtime for p in SOURCES + HEADERS)
    if not LIB.exists() or stale:
        try:
            build()
        except (OSError, EngineError) as e:
            raise EngineError(f"CUDA engine library {LIB} is {'stale' if stale else 'missing'} and could not "
                              f"be built: {e}") from e
    L = _bind(C.CDLL(str(LIB)))
    want = _header_abi_version()
    if L.fl_version() != want:
        raise EngineError(f"{LIB} has ABI version {L.fl_version()}, include/flint_b200.h {want}: rebuild it")
    _lib = L
    return _lib


def _bind(L):
    L.fl_version.restype = C.c_int
    L.fl_last_error.restype = C.c_char_p
    L.fl_device_count.argtypes = [P32]
    L.fl_graph_create.argtypes = [C.POINTER(GraphDesc), C.c_int32, C.POINTER(C.c_void_p)]
    L.fl_graph_destroy.argtypes = [C.c_void_p]
    L.fl_graph_max_nodes.argtypes = [C.c_void_p]
    L.fl_graph_max_nodes.restype = C.c_int32
    L.fl_sweep_run.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]       # (fl_points *, fl_outputs *) by address
    L.fl_sweep_run_device.argtypes = [C.c_void_p, C.POINTER(Points), C.POINTER(Outputs), C.c_void_p, P32]
    L.fl_critical_path.argtypes = [C.c_void_p, C.POINTER(Points), C.c_int32, P32, P32, P32, P32, P32, P32, P32,
                                   P32, P64, P32]
    L.fl_critical_path_values.argtypes = [C.c_void_p, C.POINTER(Points), C.c_int32, P32, P32, P32, P32, P32, P32,
                                          P32, P32, P64, P32, P64]
    L.fl_topo_order.argtypes = [C.c_void_p, P32, P32]
    L.fl_cost_only.argtypes = [C.c_int32, PU8, P64, P64, PU8, PF64, PF64, P32, P32, P64, P32,
                               C.c_int32, P64, PF64, PF64, P64]
    return L


def device_count() -> int:
    """GPUs the engine can see (0 when none; the engine then refuses to run)."""
    n = C.c_int32(0)
    lib().fl_device_count(C.byref(n))
    return int(n.value)


def last_error() -> str:
    return lib().fl_last_error().decode(errors="replace")


EXPORTED = ["fl_version", "fl_last_error", "fl_device_count", "fl_graph_create", "fl_graph_destroy",
            "fl_graph_max_nodes", "fl_sweep_run", "fl_sweep_run_device", "fl_critical_path",
            "fl_critical_path_values", "fl_cost_only", "fl_topo_order"]
