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


def _fail_at(path: str, line: int, what: str):
    raise ValidationError(f"{path}:{line}: {what}")  # dataio.cpp:18-21


def _is_unsigned(v) -> bool:
    return isinstance(v, int) and not isinstance(v, bool) and v >= 0


def _is_number(v) -> bool:
    return isinstance(v, (int, float)) and not isinstance(v, bool)


def _parse_file(path: str):
    """dataio.cpp:23-31."""
    try:
        with open(path, "r", encoding="utf-8") as f:
            text = f.read()
    except OSError:
        raise ValidationError("cannot open: " + path) from None
    try:
        return json.loads(text)
    except ValueError as e:
        raise ValidationError(f"{path}: {e}") from None


def _for_each_jsonl(path: str):
    """dataio.cpp:33-49: one JSON value per line, blank lines skipped."""
    try:
        f = open(path, "r", encoding="utf-8")
    except OSError:
        raise ValidationError("cannot open: " + path) from None
    with f:
        for line_no, line in enumerate(f, start=1):
            if not line.strip(" \t\r\n"):
                continue
            try:
                j = json.loads(line)
            except ValueError as e:
                _fail_at(path, line_no, str(e))
            yield line_no, j


def _to_attr_id(v, path: str, line: int) -> int:
    """dataio.cpp:51-58."""
    if not _is_unsigned(v):
        _fail_at(path, line, "attribute ids must be unsigned integers")
    if v > 0xFFFFFFFF:
        _fail_at(path, line, "attribute id out of range")
    return int(v)


def read_schema_json(path: str) -> IngestSchema:
    """read_schema_json (dataio.cpp:118-140)."""
    j = _parse_file(path)
    if not isinstance(j, dict) or "clauses" not in j or "dim" not in j:
        raise ValidationError(path + ": schema needs 'clauses' and 'dim'")
    names = j["clauses"]
    if not isinstance(names, list):
        raise ValidationError(path + ": 'clauses' must be an array")
    schema = IngestSchema()
    for name in names:
        if not isinstance(name, str):
            raise ValidationError(path + ": clause names must be strings")
        schema.clause_names.append(name)
    if not schema.clause_names:
        raise ValidationError(path + ": 'clauses' must not be empty")
    if not _is_unsigned(j["dim"]) or j["dim"] > 0xFFFFFFFF:
        raise ValidationError(path + ": dim must be an unsigned integer")
    schema.dim = int(j["dim"])
    return schema


def read_documents_jsonl(path: str, schema: IngestSchema) -> List[DocumentInput]:
    """read_documents_jsonl (dataio.cpp:142-187): one document per line,
    {"id": "doc1", "clauses": {"geo": [934]}, "embedding": [0.1, ...]}; an
    absent clause is empty, an absent embedding the zero vector."""
    slot_of = {n: i for i, n in enumerate(schema.clause_names)}
    docs: List[DocumentInput] = []
    for line, j in _for_each_jsonl(path):
        if not isinstance(j, dict) or not isinstance(j.get("id"), str):
            _fail_at(path, line, "document needs a string 'id'")
        clauses: List[List[int]] = [[] for _ in schema.clause_names]
        if "clauses" in j:
            cl = j["clauses"]
            if not isinstance(cl, dict):
                _fail_at(path, line, "'clauses' must be an object")
            for name, ids in cl.items():
                if name not in slot_of:
                    _fail_at(path, line, f"unknown clause '{name}'")
                if not isinstance(ids, list):
                    _fail_at(path, line, f"clause '{name}' must be an array")
                for v in ids:
                    clauses[slot_of[name]].append(_to_attr_id(v, path, line))
        if "embedding" in j:
            emb = j["embedding"]
            if not isinstance(emb, list):
                _fail_at(path, line, "'embedding' must be an array")
            if len(emb) != schema.dim:
                _fail_at(path, line, f"embedding: expected dim {schema.dim}, got {len(emb)}")
            vals = []
            for v in emb:
                if not _is_number(v):
                    _fail_at(path, line, "embedding entries must be numbers")
                vals.append(np.float32(float(v)))  # get<double>() then static_cast<float>
            embedding = np.asarray(vals, np.float32)
        else:
            embedding = np.zeros(schema.dim, np.float32)
        docs.append(DocumentInput(j["id"], clauses, embedding))
    return docs


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
    j = _parse_file(path)
    if not isinstance(j, dict) or not all(k in j for k in ("nodes", "seekerAttributes", "jobAttributes")):
        raise ValidationError(path + ": links export needs 'nodes', 'seekerAttributes' and 'jobAttributes'")
    out = LinksExport(nodes=list(j["nodes"]))
    for key, dst in (("seekerAttributes", out.seeker_attributes), ("jobAttributes", out.job_attributes)):
        m = j[key]
        if not isinstance(m, dict):
            raise ValidationError(f"{path}: '{key}' must be an object")
        for name, ids in m.items():
            if not isinstance(ids, list) or not all(_is_unsigned(v) and 0 < v <= 0xFFFFFFFF for v in ids):
                raise ValidationError(f"{path}: {key}.{name} must be an array of node ids")
            dst[name] = sorted(set(int(v) for v in ids))
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
