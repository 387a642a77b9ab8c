"""pyplot stand-in: every call is accepted; savefig writes a placeholder."""


class _Any:
    def __getattr__(self, name):
        return _Any()

    def __call__(self, *args, **kwargs):
        return _Any()

    def __iter__(self):
        return iter([_Any(), _Any()])

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


def subplots(*args, **kwargs):
    return _Any(), _Any()


rcParams = {}


def __getattr__(name):
    return _Any()
