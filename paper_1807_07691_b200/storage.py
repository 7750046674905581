"""HBM-resident store: the drop-in for ``gsmat.storage.load`` / ``Store``.

``load(directory)`` reads a store directory in the reference's persist()
format (/root/reference/pkg/src/gsmat/storage.py:203-271),
applies the same validation with the same StoreFormatError messages
(storage.py:222-271), and uploads every predicate's pair arrays to the GPU
once (the paper's "mark data that requires multiple transfer", §6.3).  The
device builds the aux-array indexes (gsm_store_finalize).

``from_store(store)`` uploads a reference in-memory ``Store`` (as built by
``gsmat.storage.build_store``) so the reference's own objects can be handed
to :func:`paper_1807_07691_b200.executor.execute` unchanged.
"""

from __future__ import annotations

import ctypes as C
import threading
import weakref
from pathlib import Path
from typing import Iterator, NamedTuple

import numpy as np

from . import _lib
from .dictionary import StoreDictionary
from .errors import StoreFormatError, UnknownPredicateError

MAGIC = "GSMAT1"
META_FILE = "meta"
STATS_FILE = "stats.tsv"


class StatEntry(NamedTuple):
    """storage.StatEntry (storage.py:100-103)."""

    cardinality: int
    distinct_subjects: int
    distinct_objects: int


class PairMatrix:
    """Host view of one predicate (read-only numpy arrays, u64 pairs).

    ``so_pairs``/``os_pairs`` are (nnz, 2) uint64 arrays in the file order
    (storage.py:74-78); the device copy lives in the gsm_store.
    """

    def __init__(self, pid: int, so: np.ndarray, os_: np.ndarray):
        self.pid = pid
        self.so = so
        self.os = os_

    @property
    def cardinality(self) -> int:
        return int(self.so.shape[0])

    @property
    def so_pairs(self) -> list[tuple[int, int]]:
        return [tuple(r) for r in self.so.tolist()]

    @property
    def os_pairs(self) -> list[tuple[int, int]]:
        return [tuple(r) for r in self.os.tolist()]


class DeviceStore:
    """A store whose predicate matrices are resident on one CUDA device."""

    def __init__(self, dictionary, matrices: dict[int, PairMatrix], stats: dict[int, StatEntry],
                 node_count: int, device: int = 0, shard: tuple[int, int] | None = None,
                 files: dict[int, tuple[Path, Path]] | None = None):
        self.dictionary = dictionary
        self.matrices = matrices
        self.stats = stats
        self.device = device
        self.node_count = int(node_count)
        self.shard = shard  # (index, count) of a sharded store, else None
        self._handle = C.c_void_p()
        self._ctx = threading.local()
        self._contexts: list[C.c_void_p] = []
        self._ctx_lock = threading.Lock()
        L = _lib.lib()
        max_pid = max(matrices) if matrices else 0
        _lib.check(L.gsm_store_create(device, self.node_count, max_pid, C.byref(self._handle)))
        self._finalizer = weakref.finalize(self, DeviceStore._release, self._handle.value,
                                           self._contexts)
        if files is not None:
            # loader fast path: the library streams the pair files itself
            pids = sorted(files)
            n = len(pids)
            so_p = (C.c_char_p * n)(*[bytes(Path(files[p][0])) for p in pids])
            os_p = (C.c_char_p * n)(*[bytes(Path(files[p][1])) for p in pids])
            nnz = (C.c_int64 * n)(*[matrices[p].cardinality for p in pids])
            _lib.check(L.gsm_store_load_files(self._handle, n, (C.c_int32 * n)(*pids), so_p, os_p, nnz))
        else:
            for pid in sorted(matrices):
                m = matrices[pid]
                so = np.ascontiguousarray(m.so, dtype=np.uint64)
                os_ = np.ascontiguousarray(m.os, dtype=np.uint64)
                _lib.check(L.gsm_store_put_predicate_shard(self._handle, pid, so.ctypes.data,
                                                           so.shape[0], os_.ctypes.data, os_.shape[0]))
        _lib.check(L.gsm_store_finalize(self._handle))

    @staticmethod
    def _release(handle, contexts) -> None:
        try:
            L = _lib.lib()
            for c in contexts:
                L.gsm_context_free(c)
            contexts.clear()
            if handle:
                L.gsm_store_free(C.c_void_p(handle))
        except Exception:  # pragma: no cover - interpreter shutdown
            pass

    # -- reference Store surface (storage.py:106-162) -----------------------
    @property
    def triple_count(self) -> int:
        return sum(m.cardinality for m in self.matrices.values())

    def matrix_for(self, pid: int) -> PairMatrix:
        try:
            return self.matrices[pid]
        except KeyError:
            raise UnknownPredicateError(pid) from None

    def triples(self) -> Iterator[tuple[int, int, int]]:
        for pid in sorted(self.matrices):
            for s, o in self.matrices[pid].so.tolist():
                yield (s, pid, o)

    # -- device side --------------------------------------------------------
    @property
    def handle(self) -> C.c_void_p:
        return self._handle

    def device_bytes(self) -> int:
        v = C.c_int64(0)
        _lib.check(_lib.lib().gsm_store_device_bytes(self._handle, C.byref(v)))
        return int(v.value)

    def context(self, arena_bytes: int = 0) -> C.c_void_p:
        """Per-thread execution context (stream + HBM arena)."""
        ctx = getattr(self._ctx, "handle", None)
        if ctx is None:
            ctx = C.c_void_p()
            _lib.check(_lib.lib().gsm_context_create(self._handle, int(arena_bytes), C.byref(ctx)))
            with self._ctx_lock:
                self._contexts.append(ctx)
            self._ctx.handle = ctx
        return ctx

    def context_pool(self, n: int, arena_bytes: int = 256 << 20) -> list[C.c_void_p]:
        """n distinct contexts (streams + arenas) for concurrent batch execution.

        Pool contexts start with a small arena (grown on demand by the
        library), so a wide pool does not reserve n full-size arenas.
        """
        with self._ctx_lock:
            pool = self.__dict__.setdefault("_pool", [])
            while len(pool) < n:
                ctx = C.c_void_p()
                _lib.check(_lib.lib().gsm_context_create(self._handle, int(arena_bytes), C.byref(ctx)))
                self._contexts.append(ctx)
                pool.append(ctx)
            return pool[:n]

    def close(self) -> None:
        self._finalizer()


def _read_pairs(path: Path, lazy: bool = False) -> np.ndarray:
    """_pairs_from_bytes (storage.py:193-200) as an (n, 2) uint64 array;
    ``lazy`` maps the file instead of reading it (the device upload streams
    the file itself, so the host copy is only paged in if a caller reads
    ``PairMatrix.so`` / ``.os``)."""
    size = path.stat().st_size
    if size % 16 != 0:
        raise StoreFormatError(f"truncated pair file {path}: {size} bytes")
    if lazy:
        if size == 0:
            return np.zeros((0, 2), dtype=np.uint64)
        return np.memmap(path, dtype="<u8", mode="r").reshape(-1, 2)
    arr = np.fromfile(path, dtype="<u8")
    return arr.reshape(-1, 2)


def shard_owner(ids: np.ndarray, node_count: int, shards: int) -> np.ndarray:
    """Owner shard of node ids: contiguous id ranges, owner(id) =
    (id - 1) * shards // node_count (the device's shard_of, gsm_exec.cu)."""
    ids = np.asarray(ids, dtype=np.uint64)
    if node_count <= 0:
        return np.zeros(ids.shape, dtype=np.int64)
    o = ((np.maximum(ids, 1) - 1) * np.uint64(shards)) // np.uint64(node_count)
    return np.minimum(o, shards - 1).astype(np.int64)


def shard_id_range(index: int, shards: int, node_count: int) -> tuple[int, int]:
    """The ids [lo, hi) that shard ``index`` owns (the inverse of
    :func:`shard_owner`: owner(id) >= i  <=>  id - 1 >= ceil(i * N / n))."""
    lo = 0 if index == 0 else -(-index * node_count // shards) + 1
    hi = (1 << 64) - 1 if index == shards - 1 else -(-(index + 1) * node_count // shards) + 1
    return lo, hi


def _key_bound(pairs: np.ndarray, key: int) -> int:
    """First row whose key column is >= key, by binary search on the mapped
    file itself (a few page reads; np.searchsorted would copy the strided
    key column, i.e. read the whole file)."""
    lo, hi = 0, pairs.shape[0]
    while lo < hi:
        mid = (lo + hi) // 2
        if int(pairs[mid, 0]) < key:
            lo = mid + 1
        else:
            hi = mid
    return lo


def _read_shard(path: Path, lo: int, hi: int) -> np.ndarray:
    """The rows of a key-sorted pair file whose key lies in [lo, hi): one
    contiguous byte range, read with a single pread."""
    mm = _read_pairs(path, lazy=True)
    a, b = _key_bound(mm, lo), _key_bound(mm, hi)
    out = np.empty((b - a, 2), dtype=np.uint64)
    if b > a:
        with open(path, "rb") as fh:
            fh.seek(16 * a)
            got = fh.readinto(memoryview(out).cast("B"))
        if got != 16 * (b - a):
            raise StoreFormatError(f"short read of {path}")
        out = out.astype("<u8", copy=False)
    return out


def load(directory: Path | str, device: int = 0, shard: tuple[int, int] | None = None) -> DeviceStore:
    """storage.load (storage.py:222-271) into device memory.

    ``shard=(i, n)`` keeps only shard i of n (SURVEY.md §8(e) sharded mode):
    the CSR rows of subjects and the CSC rows of objects whose ids fall in
    range i (:func:`shard_owner`), read as one byte range per pair file
    (:func:`_read_shard`), so a rank reads ~1/n of the store.  Validation and ``stats`` are global, so
    every shard plans a query identically."""
    if shard is not None and not (0 <= shard[0] < shard[1]):
        raise ValueError(f"bad shard {shard}")
    directory = Path(directory)
    meta_path = directory / META_FILE
    if not meta_path.exists():
        raise StoreFormatError(f"no store at {directory}: missing {META_FILE}")
    lines = meta_path.read_text(encoding="ascii").splitlines()
    if not lines or lines[0] != MAGIC:
        found = lines[0] if lines else "<empty>"
        raise StoreFormatError(f"bad magic in {meta_path}: expected {MAGIC}, found {found}")
    if len(lines) < 4:
        raise StoreFormatError(f"truncated meta file {meta_path}")
    triple_count, pred_count, node_count = (int(x) for x in lines[1:4])

    dictionary = StoreDictionary(directory)
    if dictionary.node_count != node_count:
        raise StoreFormatError(
            f"meta declares {node_count} nodes but dictionary has {dictionary.node_count}"
        )
    stats_path = directory / STATS_FILE
    if not stats_path.exists():
        raise StoreFormatError(f"missing {stats_path}")
    stats: dict[int, StatEntry] = {}
    for raw in stats_path.read_text(encoding="ascii").splitlines():
        pid_s, card, ds, do = raw.split("\t")
        stats[int(pid_s)] = StatEntry(int(card), int(ds), int(do))
    if len(stats) != pred_count:
        raise StoreFormatError(f"meta declares {pred_count} predicates but stats has {len(stats)}")

    matrices: dict[int, PairMatrix] = {}
    files: dict[int, tuple[Path, Path]] = {}
    total = 0
    for pid in stats:
        so_path = directory / f"p{pid}.so"
        os_path = directory / f"p{pid}.os"
        if not so_path.exists() or not os_path.exists():
            raise StoreFormatError(f"missing pair files for predicate {pid}")
        files[pid] = (so_path, os_path)
        so = _read_pairs(so_path, lazy=True)
        os_ = _read_pairs(os_path, lazy=True)
        if so.shape[0] != stats[pid].cardinality:
            raise StoreFormatError(
                f"{so_path}: {so.shape[0]} pairs but stats declares {stats[pid].cardinality}"
            )
        if os_.shape[0] != so.shape[0]:
            raise StoreFormatError(f"{os_path}: {os_.shape[0]} pairs but {so_path} has {so.shape[0]}")
        total += so.shape[0]
        if shard is not None:
            # the files are sorted by key, so a shard's rows are ONE byte
            # range of each file: only that range is read
            lo, hi = shard_id_range(shard[0], shard[1], node_count)
            so = _read_shard(so_path, lo, hi)
            os_ = _read_shard(os_path, lo, hi)
        matrices[pid] = PairMatrix(pid, so, os_)
    if total != triple_count:
        raise StoreFormatError(f"meta declares {triple_count} triples but store holds {total}")
    return DeviceStore(dictionary, matrices, stats, node_count, device=device, shard=shard,
                       files=files if shard is None else None)


# Reference Store objects are unhashable dataclasses: cache by id() and keep
# a weak reference to detect a recycled id.
_UPLOADED: dict[int, tuple["weakref.ref", DeviceStore]] = {}


def from_store(store, device: int = 0) -> DeviceStore:
    """Upload a reference ``gsmat.storage.Store`` (cached per store object)."""
    if isinstance(store, DeviceStore):
        return store
    hit = _UPLOADED.get(id(store))
    if hit is not None and hit[0]() is store and hit[1].device == device:
        return hit[1]
    matrices: dict[int, PairMatrix] = {}
    for pid, m in store.matrices.items():
        so = np.asarray(m.so_pairs, dtype=np.uint64).reshape(-1, 2)
        os_ = np.asarray(m.os_pairs, dtype=np.uint64).reshape(-1, 2)
        matrices[int(pid)] = PairMatrix(int(pid), so, os_)
    stats = {int(k): StatEntry(*v) for k, v in store.stats.items()}
    node_count = store.dictionary.node_count
    if matrices:
        node_count = max(node_count, int(max((int(m.so.max()) if m.so.size else 0) for m in matrices.values())))
    dev = DeviceStore(store.dictionary, matrices, stats, node_count, device=device)
    key = id(store)
    try:
        _UPLOADED[key] = (weakref.ref(store, lambda _r, k=key: _UPLOADED.pop(k, None)), dev)
    except TypeError:  # not weak-referenceable: no caching
        pass
    return dev


# -- build / persist (storage.py:165-219) -----------------------------------

class EncodedTriple(NamedTuple):
    """storage.EncodedTriple: one triple of dictionary ids."""

    s: int
    p: int
    o: int


# The reference's names for the store and its per-predicate matrices.
Store = DeviceStore
PredicateMatrix = PairMatrix


def build_store(dictionary, triples, device: int = 0) -> DeviceStore:
    """storage.build_store (storage.py:165-177): partition encoded triples by
    predicate, drop duplicates, sort both orientations and index them — the
    deduplication and sorting on the device (``gsm_sort_triples``); the
    result is already resident on ``device``."""
    rows = [tuple(t) for t in triples]
    arr = np.asarray(rows, dtype=np.uint64).reshape(-1, 3)
    if arr.size and int(arr.max()) >= 1 << 32:
        raise ValueError("ids must be < 2^32")
    s_ = np.ascontiguousarray(arr[:, 0], dtype=np.uint32)
    p_ = np.ascontiguousarray(arr[:, 1], dtype=np.uint32)
    o_ = np.ascontiguousarray(arr[:, 2], dtype=np.uint32)
    n = arr.shape[0]
    max_pid = int(p_.max()) if n else 0
    counts = (C.c_int64 * (3 * (max_pid + 1)))()
    L = _lib.lib()
    t_so, t_os = C.c_void_p(), C.c_void_p()
    _lib.check(L.gsm_sort_triples(int(device), s_.ctypes.data if n else None, p_.ctypes.data if n else None,
                                  o_.ctypes.data if n else None, n, max_pid, C.byref(t_so), C.byref(t_os),
                                  counts))

    def take(t) -> np.ndarray:
        try:
            ptr, nb = C.c_void_p(), C.c_int64()
            _lib.check(L.gsm_text_data(t, C.byref(ptr), C.byref(nb)))
            raw = C.string_at(ptr, nb.value) if nb.value else b""
        finally:
            L.gsm_text_free(t)
        return np.frombuffer(raw, dtype="<u8").reshape(-1, 2)

    so_all, os_all = take(t_so), take(t_os)
    matrices: dict[int, PairMatrix] = {}
    stats: dict[int, StatEntry] = {}
    off = 0
    for pid in range(max_pid + 1):
        card, ds, do = (int(counts[3 * pid + k]) for k in range(3))
        if card == 0:
            continue
        matrices[pid] = PairMatrix(pid, so_all[off:off + card], os_all[off:off + card])
        stats[pid] = StatEntry(card, ds, do)
        off += card
    node_count = max(int(dictionary.node_count), int(arr[:, [0, 2]].max()) if n else 0)
    return DeviceStore(dictionary, matrices, stats, node_count, device=device)


def persist(store, directory: Path | str) -> None:
    """storage.persist (storage.py:203-219): the reference's store directory
    (dictionary files, meta, stats.tsv, p<ID>.so / p<ID>.os u64 LE pairs)."""
    directory = Path(directory)
    directory.mkdir(parents=True, exist_ok=True)
    store.dictionary.save(directory)
    matrices = store.matrices
    triple_count = sum(int(np.asarray(m.so).shape[0]) for m in matrices.values())
    with open(directory / META_FILE, "w", encoding="ascii", newline="\n") as fh:
        fh.write(f"{MAGIC}\n{triple_count}\n{len(matrices)}\n{store.dictionary.node_count}\n")
    with open(directory / STATS_FILE, "w", encoding="ascii", newline="\n") as fh:
        for pid in sorted(store.stats):
            st = store.stats[pid]
            fh.write(f"{pid}\t{st.cardinality}\t{st.distinct_subjects}\t{st.distinct_objects}\n")
    for pid in sorted(matrices):
        m = matrices[pid]
        (directory / f"p{pid}.so").write_bytes(np.ascontiguousarray(m.so, dtype="<u8").tobytes())
        (directory / f"p{pid}.os").write_bytes(np.ascontiguousarray(m.os, dtype="<u8").tobytes())
