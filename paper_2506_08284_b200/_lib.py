"""ctypes binding of libsphcurl.so.

Signatures are read from the C ABI header (include/sphcurl.h), so the Python
side and the header cannot drift. There is no fallback: if the library or a
GPU is missing, every call raises.
"""

import ctypes
import os
import re

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
# SPHC_LIB: load an alternative build (tuning experiments only)
LIB_PATH = os.environ.get("SPHC_LIB") or os.path.join(HERE, "libsphcurl.so")
HEADER = os.path.join(REPO, "include", "sphcurl.h")

_CT = {"q": ctypes.c_int64, "i": ctypes.c_int, "d": ctypes.c_double,
       "p": ctypes.c_void_p}


def parse_header(path=HEADER):
    """{name: (restype, argcodes, has_stream)} for every sphc_* prototype."""
    text = open(path).read()
    text = re.sub(r"/\*.*?\*/", " ", text, flags=re.S)
    out = {}
    for m in re.finditer(r"(const\s+char\s*\*|int64_t|int)\s*(sphc_\w+)\s*\(([^)]*)\)\s*;",
                         text):
        ret, name, params = m.group(1), m.group(2), m.group(3).strip()
        codes = []
        stream = False
        if params and params != "void":
            for p in params.split(","):
                p = " ".join(p.split())
                if p.endswith("*stream") or p.endswith("* stream") or p == "void *stream":
                    stream = True
                    continue
                if "*" in p:
                    codes.append("p")
                elif p.startswith("int64_t"):
                    codes.append("q")
                elif p.startswith("double"):
                    codes.append("d")
                elif p.startswith("int"):
                    codes.append("i")
                else:
                    raise ValueError(f"unparsed parameter {p!r} in {name}")
        kind = "str" if "char" in ret else ("i64" if ret == "int64_t" else "int")
        out[name] = (kind, "".join(codes), stream)
    return out


SIGS = parse_header()

_lib = None


class LibraryMissing(RuntimeError):
    pass


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise LibraryMissing(
            f"{LIB_PATH} is not built; run __graft_entry__.build() "
            "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    for name, (ret, codes, stream) in SIGS.items():
        f = getattr(L, name)
        f.argtypes = [_CT[c] for c in codes] + ([ctypes.c_void_p] if stream else [])
        f.restype = {"str": ctypes.c_char_p, "i64": ctypes.c_int64}.get(ret, ctypes.c_int)
    _lib = L
    return L


def launch_count():
    """Kernels launched by libsphcurl so far in this process."""
    return int(lib().sphc_launch_count())


_DEV = None


def stream_handle():
    """torch's current raw CUDA stream (follows torch.cuda.stream contexts and
    graph capture) without torch.cuda.current_stream()'s per-call overhead."""
    global _DEV
    if _DEV is None:
        _DEV = torch.cuda.current_device()
    return torch._C._cuda_getCurrentRawStream(_DEV)


_FN = {}


_TENSOR = torch.Tensor


def _conv(a):
    if a is None:
        return None
    if isinstance(a, _TENSOR):
        return a.data_ptr()
    if hasattr(a, "ctypes"):      # numpy (host entry points)
        return a.ctypes.data
    return int(a)


def call(name, *args):
    """Invoke an entry point; device ones run on torch's current stream."""
    ent = _FN.get(name)
    if ent is None:
        ret, codes, stream = SIGS[name]
        ent = _FN[name] = (getattr(lib(), name), len(codes),
                           tuple(i for i, c in enumerate(codes) if c == "p"), stream)
    f, nargs, pidx, stream = ent
    if len(args) != nargs:
        raise TypeError(f"{name} takes {nargs} arguments, got {len(args)}")
    conv = list(args)
    for i in pidx:
        a = conv[i]
        if a is not None:
            conv[i] = a.data_ptr() if a.__class__ is _TENSOR else _conv(a)
    if stream:
        conv.append(torch._C._cuda_getCurrentRawStream(_DEV) if _DEV is not None
                    else stream_handle())
    rc = f(*conv)
    if rc != 0 and not (name == "sphc_host_piecewise_const" and rc == -3):
        raise RuntimeError(f"{name} failed ({rc}): {lib().sphc_last_error().decode()}")
    return rc
