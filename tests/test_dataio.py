"""Corpus ingestion: the reference's schema / JSONL corpus /
links-export formats (proj/tests/test_dataio.cpp:46-116, :197-224) parsed by
paper_2402_13435_b200.dataio and fed to the product IndexBuilder."""

from __future__ import annotations

import json

import numpy as np
import pytest

from oracle import hyre_oracle as O


@pytest.fixture(scope="module")
def dio():
    from paper_2402_13435_b200 import dataio
    return dataio


@pytest.fixture(scope="module")
def hy():
    import paper_2402_13435_b200 as hy
    return hy


def write(tmp_path, name, text):
    p = tmp_path / name
    p.write_text(text)
    return str(p)


def test_schema_file_round_trips_clause_names_and_dim(dio, tmp_path):
    s = dio.read_schema_json(write(tmp_path, "schema.json", '{"clauses": ["geo", "skill"], "dim": 4}'))
    assert s.clause_names == ["geo", "skill"] and s.dim == 4


def test_schema_errors_carry_the_file_path(dio, hy, tmp_path):
    with pytest.raises(hy.ValidationError, match="broken.json"):
        dio.read_schema_json(write(tmp_path, "broken.json", "{not json"))
    with pytest.raises(hy.ValidationError, match="'clauses' must not be empty"):
        dio.read_schema_json(write(tmp_path, "empty.json", '{"clauses": [], "dim": 4}'))
    with pytest.raises(hy.ValidationError, match="cannot open"):
        dio.read_schema_json(str(tmp_path / "missing.json"))
    with pytest.raises(hy.ValidationError, match="schema needs 'clauses' and 'dim'"):
        dio.read_schema_json(write(tmp_path, "nodim.json", '{"clauses": ["geo"]}'))
    with pytest.raises(hy.ValidationError, match="dim must be an unsigned integer"):
        dio.read_schema_json(write(tmp_path, "negdim.json", '{"clauses": ["geo"], "dim": -1}'))


def test_documents_parse_clause_maps_and_optional_embeddings(dio, tmp_path):
    path = write(tmp_path, "docs.jsonl",
                 '{"id": "doc1", "clauses": {"geo": [934, 2934], "skill": [945]}, "embedding": [1, 0]}\n'
                 "\n"  # blank lines are skipped
                 '{"id": "doc2", "clauses": {"skill": [9342]}}\n')
    docs = dio.read_documents_jsonl(path, dio.IngestSchema(["geo", "skill"], 2))
    assert len(docs) == 2
    assert docs[0].doc_id == "doc1" and docs[0].clauses == [[934, 2934], [945]]
    assert list(docs[0].embedding) == [1.0, 0.0]
    # absent clause slot -> empty; absent embedding -> zeros
    assert docs[1].clauses == [[], [9342]] and list(docs[1].embedding) == [0.0, 0.0]


def test_document_errors_name_the_offending_line(dio, hy, tmp_path):
    schema = dio.IngestSchema(["geo"], 2)
    with pytest.raises(hy.ValidationError, match=":2:"):
        dio.read_documents_jsonl(write(tmp_path, "a.jsonl", '{"id": "x", "clauses": {}}\nnope\n'), schema)
    with pytest.raises(hy.ValidationError, match="unknown clause 'salary'"):
        dio.read_documents_jsonl(write(tmp_path, "b.jsonl", '{"id": "x", "clauses": {"salary": [1]}}\n'), schema)
    with pytest.raises(hy.ValidationError, match="embedding: expected dim 2, got 3"):
        dio.read_documents_jsonl(write(tmp_path, "c.jsonl", '{"id": "x", "clauses": {}, "embedding": [1, 2, 3]}\n'),
                                 schema)
    with pytest.raises(hy.ValidationError, match="document needs a string 'id'"):
        dio.read_documents_jsonl(write(tmp_path, "d.jsonl", '{"clauses": {}}\n'), schema)
    with pytest.raises(hy.ValidationError, match="attribute ids must be unsigned integers"):
        dio.read_documents_jsonl(write(tmp_path, "e.jsonl", '{"id": "x", "clauses": {"geo": [1.5]}}\n'), schema)
    with pytest.raises(hy.ValidationError, match="attribute ids must be unsigned integers"):
        dio.read_documents_jsonl(write(tmp_path, "f.jsonl", '{"id": "x", "clauses": {"geo": [true]}}\n'), schema)
    with pytest.raises(hy.ValidationError, match="attribute id out of range"):
        dio.read_documents_jsonl(write(tmp_path, "g.jsonl", '{"id": "x", "clauses": {"geo": [4294967296]}}\n'),
                                 schema)


def test_ingested_corpus_builds_the_appendix_index(dio, tmp_path):
    # the appendix corpus (test_corpus.cpp:50-69) through the files: same
    # frozen layout as building it directly
    schema = dio.read_schema_json(write(tmp_path, "s.json", '{"clauses": ["geo", "skill"], "dim": 2}'))
    path = write(tmp_path, "docs.jsonl",
                 '{"id": "doc1", "clauses": {"geo": [934, 2934], "skill": [945, 342, 3112]}, "embedding": [1, 0]}\n'
                 '{"id": "doc2", "clauses": {"geo": [129], "skill": [9342, 234]}, "embedding": [0, 1]}\n')
    index = dio.build_index(dio.read_documents_jsonl(path, schema), schema, num_bits=16, seed=7)
    assert index.num_docs() == 2
    assert np.array(index.attributes).reshape(2, -1).tolist() == [[934, 2934, 342, 945, 3112], [129, 234, 9342, 0, 0]]
    assert np.array(index.offsets).reshape(2, -1).tolist() == [[0, 2, 5], [0, 1, 3]]


def _links_export(tmp_path):
    # the export of test_dataio.cpp:197-224, as write_links_export writes it
    doc = {"nodes": [{"id": 1, "seeker": [["t", "p1"]], "job": [["t", "q1"]], "jobs": ["j1"]},
                     {"id": 2, "seeker": [["t", "p1"]], "job": [["t", "q2"]], "jobs": ["j2", "j3"]}],
           "seekerAttributes": {"s1": [1, 2], "s2": [2]}, "jobAttributes": {"j1": [1], "j2": [2], "j3": [2]}}
    return write(tmp_path, "links.json", json.dumps(doc, indent=2))


def test_links_export_parses_into_node_id_vocabulary(dio, hy, tmp_path):
    ex = dio.read_links_export(_links_export(tmp_path))
    assert [n["id"] for n in ex.nodes] == [1, 2]
    assert ex.seeker_attributes == {"s1": [1, 2], "s2": [2]}
    assert ex.job_attributes["j3"] == [2]
    docs, schema = dio.links_documents(ex)
    assert [d.doc_id for d in docs] == ["j1", "j2", "j3"] and [d.clauses for d in docs] == [[[1]], [[2]], [[2]]]
    assert dio.seeker_query(ex, "s2").clauses[0].attribute_ids == [2]
    assert dio.seeker_query(ex, "nobody").match_all()
    with pytest.raises(hy.ValidationError, match="links export needs"):
        dio.read_links_export(write(tmp_path, "bad.json", '{"nodes": []}'))


@pytest.mark.gpu
def test_links_index_retrieves_exactly_the_reachable_jobs(dio, hy, tmp_path):
    # acceptance.cpp:708-834 (#10): a seeker's term-only query over the
    # exported link ids returns exactly the jobs its graph nodes reach, in row
    # order, on the GPU path
    ex = dio.read_links_export(_links_export(tmp_path))
    docs, schema = dio.links_documents(ex)
    index = dio.build_index(docs, schema)
    for seeker, want in (("s1", ["j1", "j2", "j3"]), ("s2", ["j2", "j3"])):
        r = hy.execute(index, hy.HybridQuery(dio.seeker_query(ex, seeker), None, 10))
        assert [index.doc_id(h.row_id) for h in r.hits] == want


def test_json_value_rules_follow_the_reference_parser(dio, hy, tmp_path):
    # nlohmann::json semantics as dataio.cpp uses them: unsigned integers only
    # for attribute ids (not 1.0, not -1, not true), any number for embedding
    # entries, escapes decoded, duplicate keys -> last wins, key order
    s = dio.IngestSchema(["geo", "skill"], 2)
    ok = write(tmp_path, "ok.jsonl",
               '{"id": "caf\\u00e9 \\ud83d\\ude00", "clauses": {"skill": [7], "geo": [4294967295, 1]},'
               ' "embedding": [-2.5e-1, 3]}\n'
               '   \t\r\n'
               '{"id": "x", "id": "y", "embedding": [1E2, -0.0]}\n')
    d = dio.read_documents_jsonl(ok, s)
    assert [x.doc_id for x in d] == ["café \U0001F600", "y"]
    assert d[0].clauses == [[4294967295, 1], [7]] and list(d[0].embedding) == [-0.25, 3.0]
    assert list(d[1].embedding) == [100.0, -0.0] and d[1].clauses == [[], []]
    for bad, msg in [('{"id": "a", "clauses": {"geo": [1.0]}}', "attribute ids must be unsigned integers"),
                     ('{"id": "a", "clauses": {"geo": [true]}}', "attribute ids must be unsigned integers"),
                     ('{"id": "a", "clauses": {"geo": [4294967296]}}', "attribute id out of range"),
                     ('{"id": "a", "embedding": [1, "2"]}', "embedding entries must be numbers"),
                     ('{"id": "a", "clauses": {"geo": 5}}', "clause 'geo' must be an array"),
                     ('{"id": "a", "clauses": []}', "'clauses' must be an object"),
                     ('{"id": 5}', "document needs a string 'id'"),
                     ('{"id": "a",}', ":1: parse error"),
                     ('{"id": "a"} x', ":1: parse error")]:
        with pytest.raises(hy.ValidationError, match=msg):
            dio.read_documents_jsonl(write(tmp_path, "bad.jsonl", bad + "\n"), s)


def test_build_index_jsonl_is_hyre_build(dio, hy, tmp_path):
    # cli_commands.cpp:37-63 in the library: widest document -> maxNumAttr
    sp = write(tmp_path, "s.json", '{"clauses": ["geo", "skill"], "dim": 2}')
    cp = write(tmp_path, "c.jsonl",
               '{"id": "doc1", "clauses": {"geo": [934, 2934], "skill": [945, 342, 3112, 945]}, "embedding": [1, 0]}\n'
               '{"id": "doc2", "clauses": {"geo": [129], "skill": [9342, 234]}, "embedding": [0, 1]}\n')
    f = dio.build_index_jsonl(sp, cp, num_bits=16, seed=7)
    assert f.max_num_attr() == 5 and f.doc_id(1) == "doc2"
    assert np.array(f.attributes)[0].tolist() == [934, 2934, 342, 945, 3112]
    with pytest.raises(hy.ValidationError, match="no documents"):
        dio.build_index_jsonl(sp, write(tmp_path, "e.jsonl", "\n"))
