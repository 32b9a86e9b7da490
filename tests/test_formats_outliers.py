"""Point-set files (BKNN binary / CSV), the outlier front end and the GPU
brute-force engine -- the behaviours the reference pins in
tests/test_datasets.py, tests/test_outliers.py and tests/test_brute.py.

CPU tests: file formats, self-match removal, scoring, ranking, and the
self-query front end driven by the CPU oracle as its engine.  GPU tests
(-m gpu): brute_knn / brute_knn_chunked / run_engine("brute") and the
B200 self-query against the oracle's brute force, bit for bit.
"""
import struct

import numpy as np
import pytest

import paper_1512_02831_b200 as bkt
from oracle import oracle as O
from paper_1512_02831_b200.datasets import FORMAT_VERSION, MAGIC

HDR = struct.Struct("<4sIQII")


def binary_file(n, d, payload=None, magic=MAGIC, version=FORMAT_VERSION):
    head = HDR.pack(magic, version, n, d, 0)
    if payload is None:
        payload = np.zeros((n, d), dtype="<f4").tobytes()
    return head + payload


def oracle_engine(refs, queries, params):
    """engine(refs, queries, params) on the CPU oracle's brute force (test side only)."""
    pm = bkt.as_point_matrix(refs)
    keys = O.brute_keys(pm.data, np.ascontiguousarray(queries, np.float32), params.k)
    return bkt.NeighborBatch.from_keys(keys, np.full(keys.shape[0], params.k, np.int64))


def oracle_outlier_scores(pts, k):
    """Mean distance to the k nearest other points, by index (float64)."""
    diff = pts[:, None, :].astype(np.float64) - pts[None, :, :]
    dd = (diff ** 2).sum(-1)
    np.fill_diagonal(dd, np.inf)
    return np.sqrt(np.sort(dd, axis=1)[:, :k]).mean(axis=1)


class TestBinary:
    def test_roundtrip_bit_exact(self, rng, tmp_path):
        pts = rng.standard_normal((37, 5)).astype(np.float32)
        bkt.write_dataset(tmp_path / "a.bknn", pts)
        back = bkt.load_dataset(tmp_path / "a.bknn")
        assert back.data.dtype == np.float32 and np.array_equal(back.data, pts)

    def test_magic_not_extension_decides(self, rng, tmp_path):
        pts = rng.random((4, 2), dtype=np.float32)
        bkt.write_dataset(tmp_path / "lies.csv", pts, fmt="binary")
        assert np.array_equal(bkt.load_dataset(tmp_path / "lies.csv").data, pts)

    def test_header_layout(self, tmp_path):
        pts = np.float32([[1.0, 2.0], [3.0, 4.0]])
        bkt.write_dataset(tmp_path / "p", pts)
        raw = (tmp_path / "p").read_bytes()
        assert raw[:24] == HDR.pack(b"BKNN", 1, 2, 2, 0)
        assert raw[24:] == pts.astype("<f4").tobytes() and len(raw) == 40

    @pytest.mark.parametrize("raw,msg", [
        (b"BKNN\x01\x00", "truncated header, 6 bytes but need 24"),
        (binary_file(1, 1, version=9), "unsupported version 9 at byte 4"),
        (binary_file(0, 3, payload=b""), "header claims 0 points of dimension 3"),
        (binary_file(3, 2)[:-4], r"payload ends at byte 44, expected 48 for 3 x 2 float32"),
    ])
    def test_malformed(self, tmp_path, raw, msg):
        (tmp_path / "p").write_bytes(raw)
        with pytest.raises(bkt.DatasetFormatError, match=msg):
            bkt.load_dataset(tmp_path / "p")

    def test_non_finite_located(self, tmp_path):
        data = np.zeros((4, 3), dtype="<f4")
        data[2, 1] = np.nan
        (tmp_path / "p").write_bytes(binary_file(4, 3, payload=data.tobytes()))
        with pytest.raises(bkt.DatasetFormatError, match="non-finite value in row 2, column 1"):
            bkt.load_dataset(tmp_path / "p")

    def test_unknown_write_format(self, rng, tmp_path):
        with pytest.raises(ValueError, match="unknown format"):
            bkt.write_dataset(tmp_path / "p", rng.random((2, 2), dtype=np.float32), fmt="json")


class TestCsv:
    def test_roundtrip(self, rng, tmp_path):
        pts = rng.standard_normal((50, 3)).astype(np.float32)
        bkt.write_dataset(tmp_path / "p.csv", pts, fmt="csv")
        assert np.array_equal(bkt.load_dataset(tmp_path / "p.csv").data, pts)

    def test_comments_and_blanks(self, tmp_path):
        (tmp_path / "p.csv").write_text("# header\n\n1.5,2.5\n\n# mid\n3.0,4.0\n")
        assert np.array_equal(bkt.load_dataset(tmp_path / "p.csv").data, np.float32([[1.5, 2.5], [3.0, 4.0]]))

    @pytest.mark.parametrize("text,msg", [
        ("1,2,3\n4,5\n", "line 2 has 2 fields, expected 3"),
        ("1,2\n3,potato\n", "line 2 is not numeric"),
        ("1,2\ninf,4\n", "non-finite value on line 2"),
        ("# only comments\n\n", "no data rows"),
    ])
    def test_malformed(self, tmp_path, text, msg):
        (tmp_path / "p.csv").write_text(text)
        with pytest.raises(bkt.DatasetFormatError, match=msg):
            bkt.load_dataset(tmp_path / "p.csv")

    def test_binary_garbage_is_an_encoding_error(self, tmp_path):
        (tmp_path / "p").write_bytes(b"\xff\xfe junk \xff")
        with pytest.raises(bkt.DatasetFormatError, match="not valid UTF-8 at byte 0"):
            bkt.load_dataset(tmp_path / "p")


class TestOutlierInstance:
    def test_planted_far_away(self):
        pts, planted = bkt.gen_outlier_instance(200, 4, 5, seed=3)
        assert planted.tolist() == sorted(planted.tolist()) and len(set(planted.tolist())) == 5
        assert (pts.data[planted] >= 3.0).all() and (np.delete(pts.data, planted, 0) < 1.0).all()

    def test_validation(self):
        with pytest.raises(ValueError):
            bkt.gen_outlier_instance(10, 2, 11)


class TestSelfMatches:
    def test_self_column_dropped_wherever_it_sits(self):
        idx = np.array([[0, 3, 2], [3, 1, 0], [2, 2, 0]], dtype=np.int64)
        sq = np.array([[0.0, 1.0, 2.0], [5.0, 0.0, 6.0], [0.0, 0.0, 7.0]], np.float32)
        ki, ks = bkt.exclude_self_matches(idx, sq)
        assert np.array_equal(ki, [[3, 2], [3, 0], [2, 0]])
        assert np.array_equal(ks, np.float32([[1, 2], [5, 6], [0, 7]]))

    def test_missing_self_drops_last_column(self):
        ki, ks = bkt.exclude_self_matches(np.array([[0, 2], [0, 2]], np.int64), np.float32([[0, 1], [0, 3]]))
        assert np.array_equal(ki, [[2], [0]]) and np.array_equal(ks, np.float32([[1], [0]]))

    def test_single_column_rejected(self):
        with pytest.raises(ValueError):
            bkt.exclude_self_matches(np.zeros((3, 1), np.int64), np.zeros((3, 1), np.float32))

    def test_rank_descending_with_index_tiebreak(self):
        assert bkt.rank_outliers(np.array([0.5, 2.0, 0.5, 1.0])).tolist() == [1, 3, 2, 0]
        assert bkt.rank_outliers(np.zeros(4)).tolist() == [3, 2, 1, 0]

    def test_scores_match_index_oracle(self, rng):
        pts = rng.random((80, 3), dtype=np.float32)
        _, sq = bkt.self_excluded_knn(bkt.PointMatrix(pts), 5, oracle_engine)
        assert np.allclose(bkt.outlier_scores(sq), oracle_outlier_scores(pts, 5), rtol=1e-6, atol=0.0)

    def test_validation(self, rng):
        pts = bkt.PointMatrix(rng.random((4, 2), dtype=np.float32))
        for k in (0, 4):
            with pytest.raises(ValueError):
                bkt.self_excluded_knn(pts, k, oracle_engine)


class TestExhaustiveStructure:
    """brute_knn's two-leaf structure with a NaN root split, checked on the
    CPU with the oracle's restatement of the reference traversal
    (kdtree.py:157-204): every query descends right (q < NaN is false) and
    visits the left leaf too ((q - NaN)^2 > kth is false), so the traversal
    is a full scan and its keys are the brute-force keys."""

    def test_traversal_is_brute_force(self, rng):
        refs = rng.random((3001, 6), dtype=np.float32)
        refs[100:140] = refs[:40]  # duplicates: ties broken by index
        q = rng.random((400, 6), dtype=np.float32)
        t = bkt.exhaustive_tree(refs)
        assert t.top.height == 1 and np.isnan(t.top.split_values[0])
        assert list(t.leaves.leaf_starts) == [0, 1500, 3001]
        ot = O.OracleTree(1, 6, t.top.split_values, np.ascontiguousarray(t.leaves.points), t.leaves.original_index,
                          t.leaves.leaf_starts)
        for k in (1, 7, 40):
            r = O.knn_tree(ot, q, k, threads=2)
            assert np.array_equal(r["keys"], O.brute_keys(refs, q, k, threads=2))
            assert np.all(r["visited"] == 2)

    def test_needs_two_points(self):
        with pytest.raises(ValueError):
            bkt.exhaustive_tree(np.zeros((1, 3), np.float32))


@pytest.mark.gpu
class TestGpuBrute:
    def test_brute_matches_oracle(self, rng, gpu_device):
        refs = rng.random((3000, 7), dtype=np.float32)
        q = rng.random((500, 7), dtype=np.float32)
        counter = bkt.EvalCounter()
        res = bkt.brute_knn(refs, q, bkt.SearchParams(k=9), counter=counter, device=gpu_device)
        assert np.array_equal(res.keys, O.brute_keys(refs, q, 9))
        assert counter.pairs == 3000 * 500

    @pytest.mark.parametrize("d,k", [(10, 10), (10, 50), (3, 1), (40, 12), (10, 100)])
    def test_brute_on_the_engine_scans(self, rng, gpu_device, d, k):
        """brute_knn runs the engine's leaf scans over an exhaustive two-leaf
        structure (tensor-core filter for d = 10, CUDA-core scan for d = 3,
        the general-domain path for d = 40 / k = 100): bit-identical to the
        oracle's brute force on a mixture with duplicated points."""
        pts, _ = bkt.gen_mixture(60_000, d, seed=d + k)
        refs = np.ascontiguousarray(pts.data[:50_000])
        refs[1000:1100] = refs[:100]  # ties broken by index
        q = np.ascontiguousarray(pts.data[50_000:])
        res = bkt.brute_knn(refs, q, bkt.SearchParams(k=k), device=gpu_device)
        assert np.array_equal(res.keys, O.brute_keys(refs, q, k, threads=O.default_threads()))

    def test_chunked_equals_single(self, rng, gpu_device):
        refs = rng.random((2501, 5), dtype=np.float32)
        q = rng.random((300, 5), dtype=np.float32)
        one = bkt.brute_knn(refs, q, bkt.SearchParams(k=4), device=gpu_device)
        many = bkt.brute_knn_chunked(refs, q, bkt.SearchParams(k=4), gpu_device, bkt.ChunkPlan.build(2501, 7))
        assert np.array_equal(one.keys, many.keys)

    def test_run_engine_brute_equals_tree(self, rng):
        refs = rng.random((4000, 6), dtype=np.float32)
        q = rng.random((700, 6), dtype=np.float32)
        a, info = bkt.run_engine("brute", refs, q, bkt.SearchParams(k=5))
        b, _ = bkt.run_engine("bufferkdtree", refs, q, bkt.SearchParams(k=5), height=4)
        assert np.array_equal(a.keys, b.keys) and info["pairs"] == 4000 * 700

    def test_self_query_on_the_tree_engine(self, rng):
        base = rng.random((900, 4), dtype=np.float32)
        pts = np.vstack([base, base[:20]])  # exact twins displace self matches
        idx, sq = bkt.self_excluded_knn(bkt.PointMatrix(pts), 6)
        ridx, rsq = bkt.self_excluded_knn(bkt.PointMatrix(pts), 6, oracle_engine)
        assert np.array_equal(sq, rsq) and np.array_equal(idx, ridx)

    def test_planted_outliers_rank_first(self):
        pts, planted = bkt.gen_outlier_instance(4000, 5, 6, seed=2)
        _, sq = bkt.self_excluded_knn(pts, 10)
        order = bkt.rank_outliers(bkt.outlier_scores(sq))
        assert set(order[:6].tolist()) == set(planted.tolist())


class TestCli:
    """The command-line front end (reference cli.py:105-177)."""

    def test_parser(self):
        from paper_1512_02831_b200 import cli
        a = cli.build_parser().parse_args(["query", "--refs", "r.bknn", "--queries", "q.bknn", "--k", "7",
                                           "--engine", "brute", "--num-chunks", "3"])
        assert (a.cmd, a.k, a.engine, a.num_chunks) == ("query", 7, "brute", 3)
        with pytest.raises(SystemExit):
            cli.build_parser().parse_args(["query", "--refs", "r.bknn", "--queries", "q", "--engine", "kdtree-cpu"])

    @pytest.mark.gpu
    def test_query_and_build_on_files(self, rng, tmp_path):
        import json
        from paper_1512_02831_b200 import cli
        refs = rng.random((5000, 6), dtype=np.float32)
        q = rng.random((700, 6), dtype=np.float32)
        bkt.write_dataset(tmp_path / "r.bknn", bkt.PointMatrix(refs))
        bkt.write_dataset(tmp_path / "q.csv", bkt.PointMatrix(q), fmt="csv")
        rep = tmp_path / "rep.json"
        assert cli.main(["query", "--refs", str(tmp_path / "r.bknn"), "--queries", str(tmp_path / "q.csv"),
                         "--k", "5", "--height", "5", "--out", str(tmp_path / "nn.npz"),
                         "--report-out", str(rep)]) == 0
        got = np.load(tmp_path / "nn.npz")
        want = O.brute_keys(refs, bkt.load_dataset(tmp_path / "q.csv").data, 5)
        wd, wi = bkt.unpack_keys(want)
        assert np.array_equal(got["indices"], wi) and np.array_equal(got["sq_dists"], wd)
        assert json.load(open(rep))["digest"] == bkt.result_digest(bkt.NeighborBatch.from_keys(want, 5))
        assert cli.main(["build", "--refs", str(tmp_path / "r.bknn"), "--height", "6", "--on-gpu"]) == 0
