"""Stream wire format (cmd_gen.cpp:39-57) through wallace_write_stream:
f64le / text / f32le, pool-major for batches, chunked with overlapped
generation/copy/write; acceptance criterion 9 (acceptance_test.cpp:391-419):
the file bytes are the in-process stream bit for bit, across runs and APIs."""
import os
import threading

import numpy as np
import pytest

import paper_1005_2314_b200 as pb
from oracle.oracle import Cfg, OracleGen, RefGen

pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("oracle_built")]


def test_criterion9_f64le_determinism(cuda, ref, tmp_path):
    cfg = dict(pool_size=1024, seed=42)
    files = []
    for k in range(2):
        b = pb.PoolBatch(pb.GeneratorConfig(**cfg), n_pools=1, seeds=[42], dtype="f64")
        f = tmp_path / f"det{k}.bin"
        b.write_stream(f, 1000000, "f64le")
        files.append(f.read_bytes())
    assert len(files[0]) == 8000000 and files[0] == files[1]
    vals = np.frombuffer(files[0], dtype="<f8")
    by_fill = RefGen(Cfg(**cfg)).fill(1000000)
    assert np.array_equal(vals.view(np.uint64), by_fill.view(np.uint64))
    g = RefGen(Cfg(**cfg))
    assert all(g.next_normal() == v for v in vals[:20000])


def test_text_format_matches_printf(cuda, tmp_path):
    cfg = dict(pool_size=256, discard_every=2, seed=7, out_mean=1.5, out_sigma=0.25)
    b = pb.PoolBatch(pb.GeneratorConfig(**cfg), n_pools=1, seeds=[7], dtype="f64")
    b.fill(33)  # a partial emission carried into the stream
    f = tmp_path / "v.txt"
    b.write_stream(f, 70000, "text")
    lines = f.read_text().splitlines()
    o = OracleGen(Cfg(**cfg), "f64")
    o.fill(33)
    want = o.fill(70000)
    assert len(lines) == 70000
    assert lines == ["%.17g" % v for v in want]
    assert np.array_equal(np.array([float(x) for x in lines]), want)  # round trip


@pytest.mark.parametrize("dtype,fmt", [("f32", "f64le"), ("f32", "f32le"), ("f64", "f64le")])
def test_multi_pool_pool_major_chunks(cuda, tmp_path, dtype, fmt):
    """16384 pools x 20000 values force several 512 MiB chunks; pool p's values land at
    [p*count, (p+1)*count) (the fill layout)."""
    kw = dict(pool_size=1024, discard_every=2)
    P, count = 16384, 20000
    seeds = np.arange(1, P + 1, dtype=np.uint64)
    b = pb.PoolBatch(pb.GeneratorConfig(**kw), n_pools=P, seeds=seeds, dtype=dtype)
    f = tmp_path / "m.bin"
    b.write_stream(f, count, fmt)
    data = np.fromfile(f, dtype="<f4" if fmt == "f32le" else "<f8")
    assert data.size == P * count
    data = data.reshape(P, count)
    for p in (0, 1, 8191, P - 1):
        want = OracleGen(Cfg(seed=int(seeds[p]), **kw), dtype).fill(count)
        want = want.astype(np.float32 if fmt == "f32le" else np.float64)
        assert np.array_equal(data[p].view(np.uint32 if fmt == "f32le" else np.uint64),
                              want.view(np.uint32 if fmt == "f32le" else np.uint64)), p
    # the stream continues after the block
    nxt = b.fill(10).cpu().numpy()
    o = OracleGen(Cfg(seed=int(seeds[5]), **kw), dtype)
    o.fill(count)
    assert np.array_equal(nxt[5], o.fill(10))


def test_pipe_and_errors(cuda):
    b = pb.PoolBatch(pb.GeneratorConfig(pool_size=128, seed=3), n_pools=1, seeds=[3], dtype="f64")
    r, w = os.pipe()
    got = bytearray()

    def reader():
        while True:
            chunk = os.read(r, 1 << 16)
            if not chunk:
                break
            got.extend(chunk)

    t = threading.Thread(target=reader)
    t.start()
    b.write_stream(w, 3000, "f64le")  # not seekable: sequential writes
    os.close(w)
    t.join()
    os.close(r)
    want = OracleGen(Cfg(pool_size=128, seed=3), "f64").fill(3000)
    assert bytes(got) == want.astype("<f8").tobytes()
    b2 = pb.PoolBatch(pb.GeneratorConfig(pool_size=128), n_pools=2, seeds=[1, 2], dtype="f64")
    with pytest.raises(pb.InvalidParameterError):
        b2.write_stream(os.devnull, 10, "text")  # several pools: binary only
    with pytest.raises(pb.InvalidParameterError):
        b2.write_stream(os.devnull, 10, "f32le")  # f32le needs an fp32 handle
