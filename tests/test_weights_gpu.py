"""MFW1 blob -> device loader (reference weights.py:142-204)
and the native transpose+cast weight packing behind it."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def eet(cuda_ok):
    import paper_2104_12470_b200 as m
    return m


@pytest.mark.parametrize("dt", [0, 1, 2])
@pytest.mark.parametrize("rows,cols", [(1, 1), (37, 70), (64, 32), (768, 2304), (1000, 33)])
def test_transpose_cast_matches_torch(eet, dt, rows, cols):
    from paper_2104_12470_b200 import _lib
    td = {0: torch.float32, 1: torch.bfloat16, 2: torch.float16}[dt]
    src = torch.randn(rows, cols, device="cuda", dtype=torch.float32)
    dst = torch.empty(cols, rows, device="cuda", dtype=td)
    _lib.call("eet_transpose_cast", dt, src.data_ptr(), rows, cols, dst.data_ptr(),
              torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert torch.equal(dst, src.t().contiguous().to(td))        # RN cast on both sides: bit-exact


@pytest.mark.parametrize("label", ["fp32", "fp16"])
def test_device_loader_generates_same_tokens(eet, tmp_path, label):
    cfg = eet.ModelConfig(batch_size=3, hidden_size=128, layer_count=2, head_count=4,
                          max_prompt=12, max_sequence=28, datatype_label=label)
    w = eet.random_weights(cfg, 96, 11)
    path = tmp_path / "w.mfw1"
    eet.save_weights(w, path)
    wd = eet.load_weights_device(path)
    assert wd.hidden_size == 128 and wd.layer_count == 2 and wd.vocab == 96
    assert wd.layers[1].w1.is_cuda and tuple(wd.layers[1].w1.shape) == (128, 512)
    assert np.array_equal(wd.layers[0].wq.cpu().numpy(), np.asarray(w.layers[0].wq))
    req = eet.GenerationRequest(prompts=[[1, 2, 3], [4, 5, 6, 7, 8, 9], [10]], steps=12)
    assert np.array_equal(eet.generate(wd, req, cfg), eet.generate(w, req, cfg))


def test_device_loader_validates_blob(eet, tmp_path):
    cfg = eet.ModelConfig(batch_size=1, hidden_size=32, layer_count=1, head_count=2,
                          max_prompt=4, max_sequence=8)
    w = eet.random_weights(cfg, 16, 3)
    path = tmp_path / "w.mfw1"
    eet.save_weights(w, path)
    raw = path.read_bytes()
    (tmp_path / "short.mfw1").write_bytes(raw[:-8])
    (tmp_path / "long.mfw1").write_bytes(raw + b"\0" * 8)
    (tmp_path / "magic.mfw1").write_bytes(b"XXXX" + raw[4:])
    for name, msg in [("short", "truncated"), ("long", "trailing"), ("magic", "bad magic")]:
        with pytest.raises(ValueError, match=msg):
            eet.load_weights_device(tmp_path / f"{name}.mfw1")
