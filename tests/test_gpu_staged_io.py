"""GPU: large copies between the device and PAGEABLE host memory go through the
context's pinned staging ring (solver.cu stage_copy: whole-row chunks of a
padded device layout, byte chunks of one long array, DMA overlapped with
multi-threaded host copies).  Results must be bit-identical to the same solve
with device-resident inputs and to writes into pinned output buffers."""
import numpy as np
import pytest
import torch

import paper_2002_12872_b200 as P
from paper_2002_12872_b200 import problems as pr

pytestmark = pytest.mark.gpu


def _np(x):
    return x.cpu().numpy() if torch.is_tensor(x) else np.asarray(x)


def _dev(p):
    dev = torch.device("cuda")
    if hasattr(p.delta, "rowptr"):
        delta = P.CsrMatrix(len(p.d), torch.as_tensor(p.delta.rowptr, device=dev),
                            torch.as_tensor(p.delta.cols, device=dev), torch.as_tensor(p.delta.vals, device=dev))
    else:
        delta = torch.as_tensor(p.delta, device=dev)
    return P.PartitionedProblem(torch.as_tensor(p.d, device=dev), delta, p.lam)


@pytest.mark.parametrize("n", [1025, 1536])  # odd n: padded device rows (2-D staged copies); even: 1-D
def test_dense_host_arrays_match_device_inputs(n):
    p, o, _ = pr.config("c1", n)
    h = P.iterate_full(p, P.IterationOptions(**o))
    d = P.iterate_full(_dev(p), P.IterationOptions(**o))
    assert int(h.status) == int(d.status) and h.iterations == d.iterations
    assert np.array_equal(h.state.a, _np(d.state.a))
    assert np.array_equal(h.eigenvalues, _np(d.eigenvalues)) and np.array_equal(h.residuals, _np(d.residuals))
    # pinned caller buffers take the direct path: same bits
    outs = (torch.empty((n, n), dtype=torch.float64, pin_memory=True).numpy(),
            torch.empty(n, dtype=torch.float64, pin_memory=True).numpy(),
            torch.empty(n, dtype=torch.float64, pin_memory=True).numpy())
    P.iterate_full(p, P.IterationOptions(**o), out=outs)
    assert np.array_equal(outs[0], h.state.a) and np.array_equal(outs[1], h.eigenvalues)


def test_csr_host_arrays_match_device_inputs():
    p, o, _ = pr.config("c4b", 300001)  # cols 19 MB, values 38 MB: several staged chunks, ragged tail
    h = P.dominant_eigenpair(p, P.IterationOptions(**o))
    d = P.dominant_eigenpair(_dev(p), P.IterationOptions(**o))
    assert int(h.status) == int(d.status) and h.iterations == d.iterations
    assert np.array_equal(h.z_chart, _np(d.z_chart)) and h.eigenvalue == d.eigenvalue


def test_dominant_selection_large_host_levels():
    """n >= 2^16 host levels are scanned on the device (temporary copy): same
    row, same ambiguity / degeneracy payloads as the host scans."""
    n = 70000
    d = np.linspace(0.0, 1.0, n)
    z = P.CsrMatrix(n, np.zeros(n + 1, dtype=np.int64), np.zeros(0, dtype=np.int32), np.zeros(0))
    r = P.dominant_eigenpair(P.PartitionedProblem(d, z, 0.5))
    assert r.row == n - 1 and r.iterations == 1 and r.eigenvalue == 1.0
    tie = d.copy()
    tie[5] = 1.0  # runner-up equal to the maximum: ambiguous, payload (first max, runner-up)
    with pytest.raises(P.DegenerateSpectrum) as e:
        P.dominant_eigenpair(P.PartitionedProblem(tie, z, 0.5))
    assert (e.value.first(), e.value.second()) == (5, n - 1)
    # same pair from the device-resident levels
    with pytest.raises(P.DegenerateSpectrum) as e2:
        P.dominant_eigenpair(P.PartitionedProblem(torch.as_tensor(tie, device="cuda"), z, 0.5))
    assert (e2.value.first(), e2.value.second()) == (5, n - 1)
    nan = d.copy()
    nan[7] = np.nan  # NaN levels take the host scans
    r = P.dominant_eigenpair(P.PartitionedProblem(nan, z, 0.5))
    assert r.row == n - 1
