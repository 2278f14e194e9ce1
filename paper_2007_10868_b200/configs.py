"""Named BASELINE.json configurations rendered in the reference generator's
architecture grammar (proj/include/polycert/gen.hpp:1-27).

Weights: gen::generate(MODEL_SEED, arch) (proj/src/gen.cpp:367-375, dyadic
draws gen.cpp:182-205). Inputs: gen::random_inputs(INPUT_SEED, n, dim)
(gen.cpp:377-392). clamp01 on; label = unique argmax of the concrete forward
pass (tools/main.cpp:86-100).
"""

MODEL_SEED = 7
INPUT_SEED = 8


def _mlp(width, depth, side=28, ch=1):
    s = f"input {side}x{side}x{ch}"
    for _ in range(depth):
        s += f"; dense {width}; relu"
    return s + "; dense 10"


def _resnet(blocks):
    s = "input 32x32x3; conv 3x3x64 s1 p1; relu"
    chans = [64, 128, 256, 512]
    for stage, (n, c) in enumerate(zip(blocks, chans)):
        for b in range(n):
            if stage > 0 and b == 0:
                s += (f"; block(conv 4x4x{c} s2 p1; relu; conv 3x3x{c} s1 p1 | "
                      f"conv 2x2x{c} s2 p0); relu")
            else:
                s += f"; block(conv 3x3x{c} s1 p1; relu; conv 3x3x{c} s1 p1 | skip); relu"
    return s + "; dense 10"


CONVBIG = ("input 32x32x3; conv 3x3x32 s1 p1; relu; conv 4x4x32 s2 p1; relu; "
           "conv 3x3x64 s1 p1; relu; conv 4x4x64 s2 p1; relu; dense 512; relu; "
           "dense 512; relu; dense 10")

EPS_MNIST = "0.026"
EPS_CIFAR = "0.00784313725490196"  # 2/255 as a decimal string

# name -> (arch, epsilon decimal string)
CONFIGS = {
    "mnist_6x100": (_mlp(100, 6), EPS_MNIST),
    "mnist_9x500": (_mlp(500, 9), EPS_MNIST),
    "cifar_convbig": (CONVBIG, EPS_CIFAR),
    "cifar_resnet18": (_resnet([2, 2, 2, 2]), EPS_CIFAR),
    "cifar_resnet34": (_resnet([3, 4, 6, 3]), EPS_CIFAR),
}
