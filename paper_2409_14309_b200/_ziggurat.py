"""Ziggurat tables of the installed numpy (the Gaussian sketch's generator).

The reference draws its Gaussian sketch with numpy's ``standard_normal``
(/root/reference/pkg/src/sketchls/sketch.py:95), numpy 2.3.5's 256-level
ziggurat (Marsaglia & Tsang) over 64-bit Philox draws.  Bit-exact entries
need numpy's own strip tables ``ki_double`` / ``wi_double`` /
``fi_double``, which are local read-only data of the static library numpy
installs (``numpy/random/lib/libnpyrandom.a``).  They are read from that
installed binary here (ar archive -> ELF64 symbol table -> .rodata), never
written out in source.
"""

from __future__ import annotations

import struct
from functools import lru_cache
from pathlib import Path

import numpy as np

# Published constants of the 256-strip normal ziggurat (Marsaglia & Tsang
# 2000): right-most strip start r and its reciprocal.
ZIGGURAT_NOR_R = 3.6541528853610087963519472518
ZIGGURAT_NOR_INV_R = 0.27366123732975827203338247596


def _libnpyrandom() -> Path:
    p = Path(np.__file__).resolve().parent / "random" / "lib" / "libnpyrandom.a"
    if not p.exists():
        raise FileNotFoundError(f"numpy static random library not found at {p}")
    return p


def _ar_member(data: bytes, want: str) -> bytes:
    if not data.startswith(b"!<arch>\n"):
        raise ValueError("not an ar archive")
    pos, longnames = 8, b""
    while pos + 60 <= len(data):
        hdr = data[pos:pos + 60]
        name = hdr[:16].decode().strip()
        size = int(hdr[48:58].decode().strip())
        body = data[pos + 60: pos + 60 + size]
        if name == "//":
            longnames = body
        else:
            if name.startswith("/") and name[1:].isdigit() and longnames:
                off = int(name[1:])
                end = longnames.index(b"/\n", off)
                name = longnames[off:end].decode()
            name = name.rstrip("/")
            if name == want:
                return body
        pos += 60 + size + (size & 1)
    raise KeyError(want)


def _elf_symbols(obj: bytes, names: tuple[str, ...]) -> dict[str, bytes]:
    if obj[:4] != b"\x7fELF" or obj[4] != 2:
        raise ValueError("expected ELF64 object")
    e_shoff, = struct.unpack_from("<Q", obj, 0x28)
    e_shentsize, e_shnum, e_shstrndx = struct.unpack_from("<HHH", obj, 0x3A)
    secs = []
    for i in range(e_shnum):
        (sh_name, sh_type, _flags, _addr, sh_offset, sh_size, sh_link, _info, _align,
         sh_entsize) = struct.unpack_from("<IIQQQQIIQQ", obj, e_shoff + i * e_shentsize)
        secs.append((sh_name, sh_type, sh_offset, sh_size, sh_link, sh_entsize))
    symtab = next(s for s in secs if s[1] == 2)  # SHT_SYMTAB
    strtab = secs[symtab[4]]
    out = {}
    for k in range(symtab[3] // symtab[5]):
        st_name, _info, _other, st_shndx, st_value, st_size = struct.unpack_from(
            "<IBBHQQ", obj, symtab[2] + k * symtab[5])
        s0 = strtab[2] + st_name
        nm = obj[s0: obj.index(b"\0", s0)].decode()
        if nm in names:
            sec = secs[st_shndx]
            out[nm] = obj[sec[2] + st_value: sec[2] + st_value + st_size]
    missing = set(names) - set(out)
    if missing:
        raise KeyError(f"symbols not found: {sorted(missing)}")
    return out


@lru_cache(maxsize=1)
def tables() -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """(ki uint64[256], wi float64[256], fi float64[256]) of the installed numpy."""
    data = _libnpyrandom().read_bytes()
    obj = _ar_member(data, "src_distributions_distributions.c.o")
    syms = _elf_symbols(obj, ("ki_double", "wi_double", "fi_double"))
    ki = np.frombuffer(syms["ki_double"], dtype="<u8").copy()
    wi = np.frombuffer(syms["wi_double"], dtype="<f8").copy()
    fi = np.frombuffer(syms["fi_double"], dtype="<f8").copy()
    if not (ki.shape == wi.shape == fi.shape == (256,)):
        raise ValueError("unexpected ziggurat table sizes")
    return ki, wi, fi
