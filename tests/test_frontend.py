"""NEXT-4 front-end (paper_1804_08378_b200/frontend.py): stack detection in torchvision graphs.

CPU: the optimizable-layer and stack counts of the paper's tbl:eval_detailkernel networks, as
reconciled in SURVEY.md Appendix A (FX graphs of torchvision 0.26 architectures, no weights),
and the structure of an optimized graph.  GPU: an optimized network equals the eager network.
"""
import pytest
import torch

torchvision = pytest.importorskip("torchvision")

# SURVEY.md Appendix A, column "ours" (the paper's Opt. column agrees for every net; its Stacks
# column has one more stack for the ResNets, App. A's reading: a separate final AvgPool stack)
APPENDIX_A = {"alexnet": (12, 8), "vgg11": (17, 10), "vgg16": (22, 15), "vgg16_bn": (35, 15),
              "densenet121": (247, 124), "densenet161": (327, 164), "resnet18": (39, 20),
              "resnet50": (104, 53), "resnet152": (308, 155)}


@pytest.mark.parametrize("net", sorted(APPENDIX_A))
def test_counts_match_appendix_a(net):
    from paper_1804_08378_b200 import frontend as fe
    d = fe.summary(getattr(torchvision.models, net)().eval())
    assert (d["opt_layers"], d["stacks"]) == APPENDIX_A[net]


def test_stack_signatures():
    """Appendix A's per-network stack lists."""
    from paper_1804_08378_b200 import frontend as fe
    sig = fe.summary(torchvision.models.alexnet().eval())["signatures"]
    assert sig == ["[relu,maxpool]"] * 2 + ["[relu]"] * 2 + ["[relu,maxpool]", "[copy]", "[relu,copy]", "[relu]"]
    sig = fe.summary(torchvision.models.resnet50().eval())["signatures"]
    assert sig[0] == "[batchnorm,relu,maxpool]"
    assert sig.count("[batchnorm,add,relu]") == 15 and sig[-1] == "[batchnorm,add,relu,avgpool]"
    assert sig.count("[batchnorm]") == 4                                  # down-sample branches
    sig = fe.summary(torchvision.models.densenet121().eval())["signatures"]
    assert sig[0] == "[batchnorm,relu,maxpool]" and sig[-1] == "[batchnorm,relu,avgpool]"
    assert sig.count("[avgpool]") == 3                                    # transition pools


def test_optimized_graph_structure():
    from paper_1804_08378_b200 import frontend as fe
    m = torchvision.models.resnet18().eval()
    gm = fe.optimize(m)
    stacks = [mod for mod in gm.modules() if isinstance(mod, fe.BrainSlugStack)]
    assert len(stacks) == 20
    called = [gm.get_submodule(n.target) for n in gm.graph.nodes if n.op == "call_module"]
    assert not any(isinstance(c, (torch.nn.BatchNorm2d, torch.nn.ReLU, torch.nn.MaxPool2d)) for c in called)
    assert sum(isinstance(c, torch.nn.Conv2d) for c in called) == 20


def test_inplace_relu_with_other_consumers_stays_eager():
    """x = conv(x); y = relu_(x); z = x + 1 -- the in-place ReLU changes x for z too, so it must
    not become a stack (which would write a new tensor)."""
    from paper_1804_08378_b200 import frontend as fe

    class M(torch.nn.Module):
        def __init__(self):
            super().__init__()
            self.conv = torch.nn.Conv2d(3, 3, 1)
            self.relu = torch.nn.ReLU(inplace=True)

        def forward(self, x):
            x = self.conv(x)
            y = self.relu(x)
            return y * 2.0 + x

    d = fe.summary(M().eval())
    assert d["signatures"] == ["[scale,add]"]   # the ReLU stays in PyTorch


def test_no_cpu_fallback():
    from paper_1804_08378_b200 import frontend as fe
    gm = fe.optimize(torchvision.models.alexnet().eval())
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        gm(torch.zeros(1, 3, 224, 224))


def test_training_model_rejected():
    from paper_1804_08378_b200 import frontend as fe
    with pytest.raises(ValueError):
        fe.optimize(torchvision.models.alexnet().train())


def _randomise_bn(m, seed):
    g = torch.Generator().manual_seed(seed)
    for mod in m.modules():
        if isinstance(mod, torch.nn.BatchNorm2d):
            C = mod.num_features
            mod.running_mean.copy_(torch.rand(C, generator=g) - 0.5)
            mod.running_var.copy_(torch.rand(C, generator=g) + 0.5)
            mod.weight.data.copy_(torch.rand(C, generator=g) + 0.5)
            mod.bias.data.copy_(torch.rand(C, generator=g) - 0.5)


@pytest.mark.gpu
@pytest.mark.parametrize("net", ["alexnet", "vgg11_bn", "resnet18", "resnet50", "densenet121"])
def test_optimized_network_matches_eager(net, cuda_dev):
    """The paper's claim at network level: the optimized network computes the same result
    (P:L72-73).  Convolutions run in cuDNN in both; the stacks run in libbrainslug.so."""
    from paper_1804_08378_b200 import frontend as fe
    torch.backends.cudnn.allow_tf32 = False
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.deterministic = True
    torch.manual_seed(0)
    m = getattr(torchvision.models, net)().eval()
    _randomise_bn(m, 1)
    m = m.cuda()
    x = torch.randn(2, 3, 224, 224, device="cuda")
    with torch.no_grad():
        ref = m(x)
        gm = fe.optimize(m)
        got = gm(x)
    torch.cuda.synchronize()
    n_stacks = sum(isinstance(mod, fe.BrainSlugStack) for mod in gm.modules())
    assert n_stacks == fe.summary(getattr(torchvision.models, net)().eval())["stacks"]
    assert got.shape == ref.shape
    scale = ref.abs().max().item()
    assert torch.allclose(got, ref, rtol=1e-4, atol=1e-4 * max(1.0, scale)), (got - ref).abs().max().item()
    with torch.no_grad():   # an empty batch goes through every stack as a no-op
        assert gm(x[:0]).shape == (0,) + tuple(ref.shape[1:])


class _Mixed(torch.nn.Module):
    """Every optimizable kind the front-end knows: BN, ReLU (module, functional, method), MaxPool,
    AvgPool, Dropout, scalar multiply, residual add, global average pool."""

    def __init__(self):
        super().__init__()
        self.conv1 = torch.nn.Conv2d(3, 8, 3, padding=1)
        self.bn = torch.nn.BatchNorm2d(8)
        self.pool = torch.nn.MaxPool2d(3, 2, 1)
        self.conv2 = torch.nn.Conv2d(8, 8, 1)
        self.avg = torch.nn.AvgPool2d(2, 2, count_include_pad=False)
        self.drop = torch.nn.Dropout(0.5)
        self.gap = torch.nn.AdaptiveAvgPool2d(1)
        self.fc = torch.nn.Linear(8, 4)

    def forward(self, x):
        x = self.pool(torch.nn.functional.relu(self.bn(self.conv1(x))))   # [BN, relu, maxpool]
        y = self.conv2(x)
        y = (y * 0.5 + x).relu()                                           # [scale, add, relu]
        y = self.gap(self.drop(self.avg(y)))                               # (continues the stack)
        return self.fc(torch.flatten(y, 1))


def test_mixed_model_stacks():
    from paper_1804_08378_b200 import frontend as fe
    d = fe.summary(_Mixed().eval())
    assert d["signatures"] == ["[batchnorm,relu,maxpool]", "[scale,add,relu,avgpool,copy,avgpool]"]
    assert d["opt_layers"] == 8   # the residual add is not a layer


@pytest.mark.gpu
def test_mixed_model_matches_eager(cuda_dev):
    from paper_1804_08378_b200 import frontend as fe
    torch.backends.cudnn.allow_tf32 = False
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.manual_seed(3)
    m = _Mixed().eval()
    _randomise_bn(m, 4)
    m = m.cuda()
    x = torch.randn(3, 3, 33, 31, device="cuda")
    with torch.no_grad():
        ref = m(x)
        got = fe.optimize(m)(x)
    assert torch.allclose(got, ref, rtol=1e-4, atol=1e-5), (got - ref).abs().max().item()


class _BroadcastAdd(torch.nn.Module):
    """relu(conv(x)) + b with b of shape (1, C, 1, 1): not a same-shape residual add."""

    def __init__(self):
        super().__init__()
        self.conv = torch.nn.Conv2d(3, 4, 1)
        self.b = torch.nn.Parameter(torch.arange(4.0).reshape(1, 4, 1, 1))

    def forward(self, x):
        return torch.relu(self.conv(x)) + self.b


class _ShapeArith(torch.nn.Module):
    """x.shape[2] * 2 is a Python int in eager mode; a stack must not break it."""

    def forward(self, x):
        k = x.shape[2] * 2
        return torch.relu(x) * 1.0 + k


def test_broadcast_add_excluded_with_example_input():
    from paper_1804_08378_b200 import frontend as fe
    m = _BroadcastAdd().eval()
    gm = fe.optimize(m, example_input=torch.zeros(2, 3, 5, 5))
    sig = [mod.signature() for mod in gm.modules() if isinstance(mod, fe.BrainSlugStack)]
    assert sig == ["[relu]"]          # the broadcasting add stays in PyTorch


def test_shape_arithmetic_excluded_with_example_input():
    from paper_1804_08378_b200 import frontend as fe
    gm = fe.optimize(_ShapeArith().eval(), example_input=torch.zeros(1, 2, 3, 3))
    sig = [mod.signature() for mod in gm.modules() if isinstance(mod, fe.BrainSlugStack)]
    assert sig == ["[relu,scale]"]    # int arithmetic and the tensor + int add stay in PyTorch


def test_scalar_stack_runs_python_semantics():
    """Without shape metadata, `x.shape[2] * 2` may be classified; it must still compute an int."""
    from paper_1804_08378_b200 import frontend as fe
    st = fe.BrainSlugStack([fe.LayerSpec("scale", alpha=2.0)], "s")
    assert st(7) == 14.0


@pytest.mark.gpu
def test_broadcast_add_operand_checked_at_run_time(cuda_dev):
    """Structural classification (no example input) turns the broadcasting add into a stack: the
    stack expands the (1, C, 1, 1) operand to the tensor's shape instead of reading past it."""
    from paper_1804_08378_b200 import frontend as fe
    torch.manual_seed(5)
    m = _BroadcastAdd().eval().cuda()
    x = torch.randn(2, 3, 5, 5, device="cuda")
    with torch.no_grad():
        ref = m(x)
        gm = fe.optimize(m)
        assert any(mod.signature() == "[relu,add]" for mod in gm.modules() if isinstance(mod, fe.BrainSlugStack))
        got = gm(x)
    torch.cuda.synchronize()
    assert torch.equal(got, ref)
    st = fe.BrainSlugStack([fe.LayerSpec("relu"), fe.LayerSpec("add", operand=1)], "bad")
    with pytest.raises(RuntimeError, match="does not broadcast"):
        st(x, torch.zeros(4, 1, 1, device="cuda"))
    with torch.no_grad():   # shape arithmetic stays an int through a classified stack
        gm2 = fe.optimize(_ShapeArith().eval())
        assert torch.equal(gm2(x), _ShapeArith()(x))
