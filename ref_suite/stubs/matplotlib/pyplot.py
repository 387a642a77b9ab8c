"""pyplot stand-in: every call is accepted; savefig writes a placeholder."""


class _Any:
    def __getattr__(self, name):
        return _Any()

    def __call__(self, *args, **kwargs):
        return _Any()

    def __iter__(self):  # `(line,) = ax.plot(...)`: one artist
        return iter([_Any()])

    def savefig(self, path, *args, **kwargs):
        savefig(path)

    def __setitem__(self, key, value):
        pass

    def __getitem__(self, key):
        return _Any()


def savefig(path, *args, **kwargs):
    if hasattr(path, "write"):
        path.write(b"placeholder figure (matplotlib absent)\n")
        return
    with open(path, "wb") as f:
        f.write(b"placeholder figure (matplotlib absent)\n")


class _Axes(_Any):
    def __init__(self, n):
        self.n = n

    def __iter__(self):  # `fig, (a, b) = plt.subplots(1, 2)`
        return iter([_Any() for _ in range(self.n)])


def subplots(nrows=1, ncols=1, *args, **kwargs):
    n = nrows * ncols
    return _Any(), (_Axes(n) if n > 1 else _Any())


rcParams = {}


def __getattr__(name):
    return _Any()
