"""Multi-device batch path on one B200: carve_batch with a
device listed several times runs one independent worker (its own contexts,
streams and copy/compute pipelines) per listed entry, all claiming chunks of
whole images from one shared atomic counter — the same code path as 2/4/8
physical GPUs, minus the PCIe links. Every output is checked against the CPU
oracle (test infrastructure) or the reference-generated C5 golden hashes.
"""
import json
import os

import numpy as np
import pytest

import oracle
import paper_2410_21207_b200 as cv

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def port():
    return oracle.port()


@pytest.fixture(scope="module")
def small_batch(port):
    # 1025 distinct images (ragged against every device count and chunk size)
    n, w, h, tw, th = 1025, 40, 24, 33, 20
    imgs = [port.make_test_image(w, h, k) for k in range(n)]
    want = [port.carve(x, tw, th) for x in imgs]
    return imgs, want, tw, th


@pytest.mark.parametrize("devices", [[0], [0, 0], [0, 0, 0], [0, 0, 0, 0]])
@pytest.mark.parametrize("pipes,chunk", [("1", "16"), ("2", "16"), ("3", "40"), (None, None)])
def test_batch_repeated_devices_match_oracle(small_batch, monkeypatch, devices, pipes, chunk):
    imgs, want, tw, th = small_batch
    if pipes:
        monkeypatch.setenv("CARVE_PIPELINES", pipes)
        monkeypatch.setenv("CARVE_PIPE_CHUNK", chunk)
    outs = cv.carve_batch(imgs, tw, th, devices=devices)
    for k, (o, w_) in enumerate(zip(outs, want)):
        assert np.array_equal(o, w_), k


def test_batch_repeated_devices_tiny_batches(port):
    # fewer images than workers: some workers find the queue empty
    for n in (1, 2, 3, 5):
        imgs = [port.make_test_image(29, 17, 100 + k) for k in range(n)]
        outs = cv.carve_batch(imgs, 21, 12, devices=[0, 0, 0, 0])
        for k in range(n):
            assert np.array_equal(outs[k], port.carve(imgs[k], 21, 12)), (n, k)


def test_batch_c5_shares_golden(monkeypatch):
    """The C5 workload (1024 x 1024x768 -> 896x768) through 4 workers on one GPU
    (256-image shares, as one rank of a 4-GPU box carves): the reference-generated
    hashes of the 8 sampled images."""
    c = json.load(open(os.path.join(GOLD, "golden.json")))["configs"]["C5"]
    n = 1024
    imgs = [cv.make_test_image(c["W"], c["H"], k) for k in range(n)]
    for devices in ([0, 0, 0, 0], [0, 0, 0, 0, 0, 0, 0, 0]):
        outs = cv.carve_batch(imgs, c["target_w"], c["target_h"], devices=devices)
        for k, s in c["samples"].items():
            assert f"{oracle.fnv1a64(outs[int(k)]):016x}" == s["output"], (len(devices), k)


@pytest.mark.parametrize("n,split,min_sub", [(128, "2", "64"), (130, "4", "32"), (64, "2", "16")])
def test_batch_device_resident_small_split(port, monkeypatch, n, split, min_sub):
    """carve_batch_device split into concurrent sub-batches below 256 images per
    sub-batch (CARVE_DEVICE_SPLIT_MIN), the per-rank share sizes of 4-8 GPUs."""
    import torch
    monkeypatch.setenv("CARVE_DEVICE_SPLIT", split)
    monkeypatch.setenv("CARVE_DEVICE_SPLIT_MIN", min_sub)
    w, h, tw, th = 45, 26, 37, 21
    imgs = [port.make_test_image(w, h, 500 + k) for k in range(n)]
    d_in = torch.from_numpy(np.stack(imgs)).cuda()
    d_out = torch.full((n, th, tw, 3), 7, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream()
    cv.carve_batch_device(d_in.data_ptr(), n, w, h, tw, th, d_out.data_ptr(), st.cuda_stream)
    st.synchronize()
    outs = d_out.cpu().numpy()
    for k in range(n):
        assert np.array_equal(outs[k], port.carve(imgs[k], tw, th)), k


def test_async_calls_then_sync_call_keep_scratch_ordered(port):
    """An asynchronous carve on a side stream followed at once by a synchronous call
    on the same thread: the library's scratch is ordered on its own stream, so the
    second call cannot overwrite buffers the first still uses."""
    import torch
    w, h, tw = 700, 300, 600
    img = port.make_test_image(w, h, 9)
    want = port.carve(img, tw)
    d_in = torch.from_numpy(img).cuda()
    d_out = torch.zeros((h, tw, 3), dtype=torch.uint8, device="cuda")
    side = torch.cuda.Stream()
    cv.carve_device(d_in.data_ptr(), w, h, tw, h, d_out.data_ptr(), None, side.cuda_stream)
    other = port.make_test_image(650, 280, 3)
    got_other = cv.carve(other, 560)  # synchronous, same thread, overlapping scratch
    side.synchronize()
    assert np.array_equal(d_out.cpu().numpy(), want)
    assert np.array_equal(got_other, port.carve(other, 560))
