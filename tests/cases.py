"""Shared parity cases (architectures in the reference generator's grammar)."""

# proj/tests/test_backsub.cpp:43-48 (kArchs) and friends
BACKSUB_ARCHS = [
    "input 1x1x6; dense 8; relu; dense 5; relu; dense 3",
    "input 5x5x1; conv 3x3x2 s1 p1; relu; conv 2x2x2 s1 p0; relu; dense 4",
    "input 4x4x2; block(conv 3x3x2 s1 p1; relu; conv 3x3x2 s1 p1 | skip); relu; dense 3",
    "input 5x5x1; conv 3x3x2 s2 p1; relu; dense 5; relu; dense 2",
]

EXTRA_ARCHS = [
    # golden CLI model (proj/tests/test_formats.cpp:67-73)
    "input 4x4x1; conv 3x3x2 s1 p1; relu; dense 3",
    # conv-sparsity case (test_backsub.cpp:159-174)
    "input 8x8x2; conv 3x3x3 s1 p1; relu; conv 3x3x2 s1 p1; relu; dense 3",
    # strided downsampling residual block (ResNet stage opener)
    "input 8x8x2; conv 3x3x4 s1 p1; relu; block(conv 4x4x4 s2 p1; relu; conv 3x3x4 s1 p1 | conv 2x2x4 s2 p0); relu; dense 5",
    # two residual blocks, second nested with a strided opener
    "input 8x8x3; conv 3x3x4 s1 p1; relu; block(conv 3x3x4 s1 p1; relu; conv 3x3x4 s1 p1 | skip); relu; "
    "block(conv 4x4x6 s2 p1; relu; conv 3x3x6 s1 p1 | conv 2x2x6 s2 p0); relu; block(conv 3x3x6 s1 p1; relu; conv 3x3x6 s1 p1 | skip); relu; dense 4",
    # nested join inside a branch
    "input 6x6x2; conv 3x3x3 s1 p1; relu; block(block(conv 3x3x3 s1 p1; relu | skip); relu; conv 3x3x3 s1 p1 | skip); relu; dense 3",
    # dense branch inside a block (densify path)
    "input 1x1x5; dense 6; relu; block(dense 6; relu; dense 6 | skip); relu; dense 3",
    # conv after a dense layer on a 1x1 grid, asymmetric windows
    "input 5x5x1; conv 3x3x2 s2 p0; relu; conv 2x2x3 s1 p0; relu; dense 3",
    # 1x1 convolutions and a relu target over a join
    "input 7x7x2; conv 1x1x3 s1 p0; relu; block(conv 3x3x3 s1 p1 | skip); relu; conv 3x3x2 s2 p1; relu; dense 2",
    # MLP of the MNIST family, small
    "input 4x4x1; dense 20; relu; dense 20; relu; dense 20; relu; dense 10",
    # wide channels (>= 32: the shared-memory conv kernel), strided residual block
    "input 8x8x3; conv 3x3x32 s1 p1; relu; block(conv 4x4x40 s2 p1; relu; conv 3x3x40 s1 p1 | conv 2x2x40 s2 p0); relu; conv 3x3x36 s1 p1; relu; dense 5",
]
