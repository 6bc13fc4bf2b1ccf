"""Corpus ingestion feeding the index build.

The reference's `hyre build` reads a schema file and a JSONL corpus
(`dataio.cpp:118-187`, formats in `dataio.hpp:15-28`) and the link learner's
serving-graph export (`dataio.cpp:253-274`, `link_learner.cpp:327-347`), whose
node ids become the config-5 term vocabulary: a job's attributes are the ids
of the graph nodes that reach it, a seeker's query is the ids of its nodes.
This module parses the same files with the same validation and error texts
("<path>:<line>: <what>", ValidationError) and hands the documents to the
product IndexBuilder; everything after that is the B200 path.

Host-side parsing only (the reference parses on the host too); JSON number
semantics follow nlohmann::json as the reference uses it: attribute ids must
be unsigned integers (not floats, not booleans), embedding entries any number.
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from .hyre import (CnfClause, CnfQuery, DocumentInput, FrozenIndex, IndexBuilder, IndexConfig, ValidationError,
                   make_codec)


@dataclass
class IngestSchema:
    """`IngestSchema` (dataio.hpp:15-21): {"clauses": ["geo", "skill"], "dim": 4}."""
    clause_names: List[str] = field(default_factory=list)
    dim: int = 0


def _lib():
    from . import _lib as L
    return L


def _check(rc: int) -> None:
    from .hyre import _check as check
    check(rc)


def read_schema_json(path: str) -> IngestSchema:
    """read_schema_json (dataio.cpp:118-140), parsed by the library's C++
    ingestion (csrc/ingest.cpp, hyre_schema_read_json)."""
    L = _lib()
    h = L.C.c_void_p()
    _check(L.lib().hyre_schema_read_json(path.encode(), L.C.byref(h)))
    try:
        n = L.lib().hyre_schema_num_clauses(h)
        return IngestSchema([L.lib().hyre_schema_clause_name(h, i).decode() for i in range(n)],
                            int(L.lib().hyre_schema_dim(h)))
    finally:
        L.lib().hyre_schema_destroy(h)


class _Schema:
    """An IngestSchema as a library handle (hyre_schema_create)."""

    def __init__(self, schema: IngestSchema):
        L = _lib()
        names = (L.C.c_char_p * max(1, len(schema.clause_names)))(*[n.encode() for n in schema.clause_names])
        self.h = L.C.c_void_p()
        _check(L.lib().hyre_schema_create(len(schema.clause_names), names, schema.dim, L.C.byref(self.h)))

    def __del__(self):
        if getattr(self, "h", None):
            _lib().lib().hyre_schema_destroy(self.h)


class DocumentSet:
    """read_documents_jsonl's documents held by the library (flat arrays, file
    order); `widest` is hyre build's maxNumAttr."""

    def __init__(self, path: str, schema: IngestSchema):
        L = _lib()
        self._schema = _Schema(schema)
        self.h = L.C.c_void_p()
        _check(L.lib().hyre_documents_read_jsonl(path.encode(), self._schema.h, L.C.byref(self.h)))
        self.num_clauses, self.dim = len(schema.clause_names), schema.dim

    def __del__(self):
        if getattr(self, "h", None):
            _lib().lib().hyre_documents_destroy(self.h)

    def __len__(self) -> int:
        return int(_lib().lib().hyre_documents_count(self.h))

    @property
    def widest(self) -> int:
        return int(_lib().lib().hyre_documents_widest(self.h))

    def documents(self) -> List[DocumentInput]:
        L = _lib()
        lib, n, C = L.lib(), len(self), self.num_clauses
        so = np.ctypeslib.as_array(lib.hyre_documents_slot_offsets(self.h), (n * C + 1,)) if n else np.zeros(1, np.uint64)
        ids = np.ctypeslib.as_array(lib.hyre_documents_ids(self.h), (max(1, int(so[-1])),)) if so[-1] else np.zeros(0, np.uint32)
        emb = np.ctypeslib.as_array(lib.hyre_documents_embeddings(self.h), (max(1, n * self.dim),)) if n and self.dim \
            else np.zeros(0, np.float32)
        out = []
        for i in range(n):
            cl = [ids[int(so[i * C + c]):int(so[i * C + c + 1])].tolist() for c in range(C)]
            out.append(DocumentInput(lib.hyre_documents_id(self.h, i).decode(), cl,
                                     np.array(emb[i * self.dim:(i + 1) * self.dim], np.float32)))
        return out

    def add_to(self, builder: IndexBuilder) -> int:
        """add_document for every document (file order) -> first row."""
        L = _lib()
        first = L.C.c_uint32()
        _check(L.lib().hyre_builder_add_document_set(builder._h, self.h, L.C.byref(first)))
        return int(first.value)


def read_documents_jsonl(path: str, schema: IngestSchema) -> List[DocumentInput]:
    """read_documents_jsonl (dataio.cpp:142-187): one document per line,
    {"id": "doc1", "clauses": {"geo": [934]}, "embedding": [0.1, ...]}; an
    absent clause is empty, an absent embedding the zero vector (parsed by
    csrc/ingest.cpp)."""
    return DocumentSet(path, schema).documents()


def build_index(docs: Sequence[DocumentInput], schema: IngestSchema, max_num_attr: Optional[int] = None,
                num_bits: int = 512, seed: int = 1) -> FrozenIndex:
    """`hyre build` (cli_commands.cpp:37-63): IndexConfig from the schema,
    max_num_attr = the widest document (deduplicated per clause) unless given,
    every document staged, frozen with make_codec(dim, num_bits, seed)."""
    if not docs:
        raise ValidationError("no documents")
    width = max_num_attr
    if width is None:
        width = max([sum(len(set(c)) for c in d.clauses) for d in docs] + [1])
    b = IndexBuilder(IndexConfig(len(schema.clause_names), width, schema.dim, list(schema.clause_names)))
    for d in docs:
        b.add_document(d)
    return b.freeze(make_codec(schema.dim, num_bits, seed))


def build_index_jsonl(schema_path: str, corpus_path: str, num_bits: int = 512, seed: int = 1,
                      device: Optional[int] = None) -> FrozenIndex:
    """`hyre build` (cli_commands.cpp:37-63) end to end in the library:
    schema + JSONL corpus parsed in C++, maxNumAttr = the widest document,
    every document staged, frozen (on GPU `device` if given)."""
    schema = read_schema_json(schema_path)
    ds = DocumentSet(corpus_path, schema)
    if len(ds) == 0:
        raise ValidationError("no documents")
    b = IndexBuilder(IndexConfig(len(schema.clause_names), max(1, ds.widest), schema.dim, list(schema.clause_names)))
    ds.add_to(b)
    return b.freeze(make_codec(schema.dim, num_bits, seed), device=device)


# ---------------------------------------------------------------------------
# learned-link export (config-5 vocabulary)
# ---------------------------------------------------------------------------
@dataclass
class LinksExport:
    """The serving-graph export written by write_links_export
    (dataio.cpp:253-274): nodes [{"id": i + 1, "seeker": [[attr, value]...],
    "job": [...], "jobs": [job ids]}], "seekerAttributes": {seeker: [node
    ids]}, "jobAttributes": {job: [node ids]} (export_to_index,
    link_learner.cpp:327-347)."""
    nodes: List[dict] = field(default_factory=list)
    seeker_attributes: Dict[str, List[int]] = field(default_factory=dict)
    job_attributes: Dict[str, List[int]] = field(default_factory=dict)


def read_links_export(path: str) -> LinksExport:
    """The serving-graph export (validated and mapped by csrc/ingest.cpp,
    hyre_links_read_json); `nodes` keeps the raw node records."""
    L = _lib()
    h = L.C.c_void_p()
    _check(L.lib().hyre_links_read_json(path.encode(), L.C.byref(h)))
    try:
        out = LinksExport()
        for side, dst in ((0, out.seeker_attributes), (1, out.job_attributes)):
            for i in range(L.lib().hyre_links_count(h, side)):
                n = L.C.c_uint32()
                p = L.lib().hyre_links_ids(h, side, i, L.C.byref(n))
                dst[L.lib().hyre_links_name(h, side, i).decode()] = \
                    np.ctypeslib.as_array(p, (n.value,)).tolist() if n.value else []
    finally:
        L.lib().hyre_links_destroy(h)
    with open(path, "r", encoding="utf-8") as f:
        out.nodes = list(json.load(f)["nodes"])
    return out


def links_documents(export: LinksExport, dim: int = 4,
                    embeddings: Optional[Dict[str, Sequence[float]]] = None,
                    jobs: Optional[Sequence[str]] = None) -> Tuple[List[DocumentInput], IngestSchema]:
    """One document per job with a single clause "link" holding the node ids
    that reach it (the term index of acceptance #10, acceptance.cpp:708-834).
    Jobs default to the export's jobAttributes in key order; embeddings
    optional (zero vectors: term-only retrieval)."""
    schema = IngestSchema(["link"], dim)
    names = list(jobs) if jobs is not None else list(export.job_attributes)
    docs = []
    for name in names:
        emb = np.zeros(dim, np.float32) if not embeddings or name not in embeddings else \
            np.asarray(embeddings[name], np.float32)
        docs.append(DocumentInput(name, [list(export.job_attributes.get(name, []))], emb))
    return docs, schema


def seeker_query(export: LinksExport, seeker: str) -> CnfQuery:
    """The seeker's clause over the link slot: its node ids (an unknown seeker
    or one without nodes gives the empty CNF, i.e. match-all, exactly as an
    empty clause map does in normalize_query)."""
    ids = export.seeker_attributes.get(seeker, [])
    return CnfQuery([CnfClause(0, list(ids))]) if ids else CnfQuery()
