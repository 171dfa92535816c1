"""Out-of-bounds write checks for every kernel family (a memcheck stand-in:
compute-sanitizer is closed on the GPU pool).  Input, output and workspace
live inside larger buffers whose guard bands are filled with a sentinel
pattern; after each run the bands must be untouched, the input unmodified,
and the result still correct.  Shapes are chosen so TMA boxes, pencils,
cells and tiles end exactly at (and, ragged, short of) the buffer ends."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import oracle as O  # noqa: E402

pytestmark = pytest.mark.gpu
GUARD = 1 << 16  # bytes on each side
PAT = 0x5A


def _guarded(nbytes, fill=None):
    buf = torch.full((GUARD + nbytes + GUARD,), PAT, dtype=torch.uint8, device="cuda")
    body = buf[GUARD:GUARD + nbytes]
    if fill is not None:
        body.copy_(fill)
    return buf, body


def _intact(buf, nbytes):
    head = buf[:GUARD]
    tail = buf[GUARD + nbytes:]
    return bool((head == PAT).all()) and bool((tail == PAT).all())


CASES = [
    ("4d-mdict", (64, 64, 32, 32), (8, 8, 4, 4), 256, 0.02, True, "4d"),
    ("l4d-global-mdict", (32, 64, 32, 32), (8, 8, 4, 8), 512, 0.01, False, "l4d"),
    ("5d-nb", (16, 16, 16, 16, 16), (4, 4, 2, 4, 4), 128, 0.03, True, "5d"),
    ("3d-global", (40, 48, 64), (8, 8, 8), 256, 0.02, False, "3d"),
    ("ragged-3d", (37, 29, 45), (8, 7, 6), 64, 0.05, True, None),
    ("f64-4d", (24, 20, 12, 16), (6, 5, 4, 4), 64, 0.05, True, None),
    ("rank6", (5, 4, 6, 3, 4, 5), (2, 3, 2, 2, 3, 2), 16, 0.2, False, None),
]


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_no_write_outside_buffers(case):
    import paper_1906_11355_b200 as M
    from paper_1906_11355_b200 import datasets
    name, shape, kernel, nb, clip, ad, gen = case
    if gen:
        x = datasets.make(gen, seed=9, shape=shape).numpy()
    else:
        rng = np.random.default_rng(9)
        x = np.round(rng.random(shape) * 40) / 40
        x = x.astype(np.float64 if name.startswith("f64") else np.float32)
    xt = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    code = 1 if x.dtype == np.float64 else 0
    plan = M.Plan(x.shape, kernel, nb, clip, ad, code)
    nbytes = xt.numel() * xt.element_size()
    ibuf, ibody = _guarded(nbytes, xt.view(-1).view(torch.uint8))
    obuf, obody = _guarded(nbytes)
    wbuf, wbody = _guarded(plan.workspace_bytes)
    xin = ibody.view(xt.dtype).view(xt.shape)
    out = obody.view(xt.dtype).view(xt.shape)
    for _ in range(2):  # second run: workspace reuse
        plan.enqueue(xin, out, wbody)
        plan.check(wbody)
    torch.cuda.synchronize()
    assert _intact(ibuf, nbytes) and _intact(obuf, nbytes) and _intact(wbuf, plan.workspace_bytes)
    assert torch.equal(xin, xt), "input modified"
    got = out.cpu().numpy().astype(np.float64)
    assert np.max(np.abs(got - O.mclahe(x, kernel, nb, clip, ad, "c"))) <= 1e-5
