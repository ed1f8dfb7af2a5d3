"""Synthetic model manifests: ordered key sizes (fp32 element counts).

A *key* is one layer's parameter array ("we use key to refer
to a layer").  The paper publishes only total model sizes
(Table 5, "MB" read as MiB -- DESIGN.md reading R8); the per-key
structure below follows the MXNet reference symbols named in SURVEY.md App. A
and reproduces Table 5 within 0.2%:

    AlexNet 194.0 MiB, VGG-19 548.0 MiB, ResNet-50 97.5 MiB,
    ResNet-269 389.4 MiB, ResNet-18 44.6 MiB.

The tiny parameter-server config is BASELINE.json configs[0]:
"3 keys (4 KB, 100 KB, 1 MB fp32)" read as KiB -> [1024, 25600, 262144].
"""
from __future__ import annotations


def _alexnet():
    # MXNet AlexNet symbol, 224x224 input, pool5 -> 5x5 (6x5x5x256 = 6400)
    keys = []
    convs = [(3, 96, 11), (96, 256, 5), (256, 384, 3), (384, 384, 3), (384, 256, 3)]
    for cin, cout, k in convs:
        keys += [cout * cin * k * k, cout]
    for fin, fout in [(6400, 4096), (4096, 4096), (4096, 1000)]:
        keys += [fin * fout, fout]
    return keys


def _vgg19():
    keys = []
    chans = [64, 64, 128, 128, 256, 256, 256, 256] + [512] * 8
    cin = 3
    for c in chans:
        keys += [c * cin * 9, c]
        cin = c
    for fin, fout in [(25088, 4096), (4096, 4096), (4096, 1000)]:
        keys += [fin * fout, fout]
    return keys


def _resnet_bottleneck(units):
    # MXNet pre-activation resnet.py, bottleneck units, no conv bias,
    # BatchNorm gamma and beta as separate keys.
    keys = [3, 3, 64 * 3 * 7 * 7, 64, 64]          # bn_data, conv0, bn0
    filters = [256, 512, 1024, 2048]
    cin = 64
    for f, n in zip(filters, units):
        for u in range(n):
            q = f // 4
            keys += [cin, cin, q * cin, q, q, q * q * 9, q, q, f * q]
            if u == 0:
                keys += [f * cin]                    # projection shortcut
            cin = f
    keys += [2048, 2048, 1000 * 2048, 1000]          # bn1, fc weight, fc bias
    return keys


def _resnet18():
    # basic blocks [2,2,2,2], pre-activation, no conv bias
    keys = [3, 3, 64 * 3 * 7 * 7, 64, 64]
    filters = [64, 128, 256, 512]
    cin = 64
    for si, f in enumerate(filters):
        for u in range(2):
            keys += [cin, cin, f * cin * 9, f, f, f * f * 9]
            if u == 0 and (si > 0):
                keys += [f * cin]
            cin = f
    keys += [512, 512, 1000 * 512, 1000]
    return keys


MANIFESTS = {
    "tiny": lambda: [1024, 25600, 262144],
    "resnet50": lambda: _resnet_bottleneck([3, 4, 6, 3]),
    "alexnet": _alexnet,
    "vgg19": _vgg19,
    "resnet269": lambda: _resnet_bottleneck([3, 30, 48, 8]),
    "resnet18": _resnet18,
}

# BASELINE.json configs -> (manifest name, workers N, chunk bytes)
CONFIGS = {
    "tiny": ("tiny", 4, 32768),
    "resnet50": ("resnet50", 8, 32768),
    "alexnet": ("alexnet", 8, 32768),
    "vgg19": ("vgg19", 8, 32768),
    "resnet269": ("resnet269", 8, 32768),
}

# BASELINE.json configs[4]: ResNet-269 chunk-size sweep 4 KB .. 1 MB
SWEEP_CHUNK_BYTES = [4096 << i for i in range(9)]


def manifest(name: str) -> list[int]:
    """Key sizes (fp32 elements), key order = key_id."""
    return list(MANIFESTS[name]())


def config_names() -> list[str]:
    return list(CONFIGS)
