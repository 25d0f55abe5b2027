"""The reference's .mlra checkpoint -> device.

  reference (checkpoint.hpp)                  here (libmlra C ABI, host C++)
  -----------------------------------------   ------------------------------------------------
  load_model(path) parse + validation         Checkpoint.load: same checks, same FormatError
  (checkpoint.cpp:141-306)                    kinds and byte offsets, IoError
  save_model(model, path) (:93-130, :307-314) Checkpoint.save: byte-identical re-encoding
  inspect_layout(path) (:320-322)             Checkpoint.layout()
  ToyModel::frozen_state_hash (model.cpp:203) Checkpoint.frozen_hash(); fnv1a64 file digest
  assemble_model (model.cpp:472-531)          load_model: the same structural checks
                                              (ConfigError); to_layers() takes strategy and
                                              bias_trainable from the config JSON

Each layer's packed words go to HBM verbatim (``upload``): at LLaMA shapes the
reference bitstream already is the device layout.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List, Optional

import numpy as np
import torch

from . import _lib
from ._lib import MlraError, check, lib
from .modulora import (DeviceQuantizedMatrix, LoraAdapter, MaterializationStrategy, ModuLoraLayer,
                       _stream_ptr)


def _arr(ptr, n, dt):
    if n == 0:
        return np.zeros(0, dt)
    return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(np.ctypeslib.as_ctypes_type(dt))),
                                 shape=(n,)).copy()


@dataclass
class LayerRecord:
    """One layer record with its adapter (checkpoint.hpp:11-24)."""
    name: str
    rows: int
    cols: int
    bits: int
    group_size: int
    words: np.ndarray
    scales: np.ndarray
    zeros: np.ndarray
    bias: np.ndarray
    rank: int
    alpha: float
    a: np.ndarray  # f64 [rows x rank]
    b: np.ndarray  # f64 [cols x rank]
    offset: int
    size: int
    adapter_offset: int
    adapter_size: int


class Checkpoint:
    def __init__(self, handle: C.c_void_p):
        self._h = handle

    @classmethod
    def load(cls, path: str) -> "Checkpoint":
        h = C.c_void_p()
        check(lib().mlra_checkpoint_load(path.encode(), C.byref(h)))
        return cls(h)

    def __del__(self):
        try:
            if getattr(self, "_h", None) is not None and self._h.value and _lib._lib is not None:
                lib().mlra_checkpoint_free(self._h)
                self._h = C.c_void_p()
        except Exception:
            pass

    def __len__(self) -> int:
        return int(lib().mlra_checkpoint_layer_count(self._h))

    def config_json(self) -> str:
        v = C.c_int()
        return lib().mlra_checkpoint_config_json(self._h, C.byref(v)).decode()

    def version(self) -> int:
        v = C.c_int()
        lib().mlra_checkpoint_config_json(self._h, C.byref(v))
        return v.value

    def layer(self, i: int) -> LayerRecord:
        o = _lib.MlraCkptLayer()
        check(lib().mlra_checkpoint_layer(self._h, i, C.byref(o)))
        ng = o.rows * (o.cols // o.group_size)
        return LayerRecord(
            o.name.decode(), o.rows, o.cols, o.bits, o.group_size,
            _arr(o.words, o.word_count, np.uint32), _arr(o.scales, ng, np.float32),
            _arr(o.zeros, ng, np.float32), _arr(o.bias, o.rows, np.float32), o.rank, o.alpha,
            _arr(o.a, o.rows * o.rank, np.float64).reshape(o.rows, o.rank),
            _arr(o.b, o.cols * o.rank, np.float64).reshape(o.cols, o.rank),
            o.record_offset, o.record_size, o.adapter_offset, o.adapter_size)

    def layers(self) -> List[LayerRecord]:
        return [self.layer(i) for i in range(len(self))]

    def layout(self) -> dict:
        """inspect_layout (checkpoint.cpp:320-322): record offsets and sizes; the
        adapters in adapter-section (file) order."""
        recs = self.layers()
        ads = []
        for i in range(int(lib().mlra_checkpoint_adapter_count(self._h))):
            name, off, size = C.c_char_p(), C.c_uint64(), C.c_uint64()
            check(lib().mlra_checkpoint_adapter(self._h, i, C.byref(name), C.byref(off),
                                                C.byref(size)))
            ads.append((name.value.decode(), off.value, size.value))
        return {"version": self.version(),
                "layers": [(r.name, r.offset, r.size) for r in recs], "adapters": ads}

    def config(self) -> dict:
        """The model config JSON (model_config_from_json, model.cpp:123-166)."""
        import json
        try:
            return json.loads(self.config_json())
        except ValueError as e:
            raise MlraError(3, f"model config: invalid JSON: {e}") from None

    def assemble_check(self) -> None:
        """assemble_model's structural checks (model.cpp:472-531) -> ConfigError."""
        kind = self.config().get("kind", "mlp")
        if kind not in ("mlp", "parity_transformer"):
            raise MlraError(3, f"unknown model kind '{kind}' (expected mlp or parity_transformer)")
        check(lib().mlra_checkpoint_assemble_check(self._h, int(kind == "parity_transformer")))

    def frozen_hash(self) -> int:
        return int(lib().mlra_checkpoint_frozen_hash(self._h))

    def file_hash(self) -> int:
        return int(lib().mlra_checkpoint_file_hash(self._h))

    def upload(self, i: int, stream: Optional[torch.cuda.Stream] = None) -> DeviceQuantizedMatrix:
        """Layer i's packed words + grids to HBM, verbatim (mlra_checkpoint_upload)."""
        rec = self.layer(i)
        h = C.c_void_p()
        check(lib().mlra_checkpoint_upload(self._h, i, _stream_ptr(stream), C.byref(h)))
        return DeviceQuantizedMatrix._wrap(h, rec.rows, rec.cols, rec.bits, rec.group_size)

    def to_layers(self, strategy=None, bias_trainable=None) -> List[ModuLoraLayer]:
        """Device ModuLoraLayers as assemble_model builds them (model.cpp:508-531):
        frozen weights uploaded, bias and adapter factors as fp32 device tensors
        (the f64 values stay available through layer(i).a / .b for an exact AdamW
        master copy); strategy and bias_trainable from the config JSON unless
        given explicitly."""
        from .modulora import parse_strategy
        self.assemble_check()
        cfg = self.config()
        if strategy is None:
            strategy = parse_strategy(cfg.get("strategy", "row"))
        if bias_trainable is None:
            bias_trainable = bool(cfg.get("bias_trainable", False))
        out = []
        for i in range(len(self)):
            r = self.layer(i)
            ad = LoraAdapter(torch.from_numpy(r.a.astype(np.float32)).cuda(),
                             torch.from_numpy(r.b.astype(np.float32)).cuda(), r.rank, float(r.alpha))
            out.append(ModuLoraLayer(r.name, self.upload(i), ad,
                                     bias=torch.from_numpy(r.bias).cuda(),
                                     bias_trainable=bool(bias_trainable),
                                     strategy=MaterializationStrategy(strategy)))
        return out

    def set_adapter(self, i: int, a: np.ndarray, b: np.ndarray) -> None:
        rec = self.layer(i)
        a = np.ascontiguousarray(a, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        if a.shape != (rec.rows, rec.rank) or b.shape != (rec.cols, rec.rank):
            raise MlraError(2, "checkpoint: adapter shape mismatch")
        check(lib().mlra_checkpoint_set_adapter(self._h, i, a.ctypes.data, b.ctypes.data))

    def save(self, path: str) -> None:
        check(lib().mlra_checkpoint_save(self._h, path.encode()))


def load_model(path: str) -> Checkpoint:
    """load_model (checkpoint.cpp:324-327): parse + validation (FormatError / IoError),
    then assemble_model's checks (ConfigError)."""
    c = Checkpoint.load(path)
    c.assemble_check()
    return c


def inspect_layout(path: str) -> dict:
    return Checkpoint.load(path).layout()
