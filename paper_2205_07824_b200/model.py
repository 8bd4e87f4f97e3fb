"""PDE model descriptions consumed by the LDG hot path.

Host-side setup restated from ``ldgkit/model.py`` so models can be built on
a machine without the reference package: the same ``PdeModel`` attributes
and plan accessors (``model.py:116-218``), the builtin library
(``model.py:567-752``) and the sectioned model-file grammar
(``model.py:317-497``).  A reference ``PdeModel`` can be passed anywhere a
model from this module is accepted.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .expr import ExprSyntaxError, compile_texts, parse_expression

KINDS = ("C", "D", "W")
BC_TYPES = ("dirichlet", "neumann", "absorbing", "periodic")


class ModelError(ValueError):
    pass


class ModelFileError(ModelError):
    def __init__(self, message, line=None):
        super().__init__(message + ("" if line is None else f" (line {line})"))
        self.line = line


def reserved_symbols(ncu, nd, nw, nparam):
    """Symbol table order (model.py:48-57)."""
    s = [f"x{k}" for k in range(1, nd + 1)] + ["t"]
    s += [f"u{i}" for i in range(1, ncu + 1)]
    s += [f"q{i}_{j}" for i in range(1, ncu + 1) for j in range(1, nd + 1)]
    s += [f"w{i}" for i in range(1, nw + 1)]
    s += [f"mu{i}" for i in range(1, nparam + 1)]
    s += [f"n{k}" for k in range(1, nd + 1)]
    return tuple(s)


def face_symbols(ncu, nd, nparam):
    s = [f"x{k}" for k in range(1, nd + 1)] + ["t"]
    s += [f"ul{i}" for i in range(1, ncu + 1)]
    s += [f"ur{i}" for i in range(1, ncu + 1)]
    s += [f"ql{i}_{j}" for i in range(1, ncu + 1) for j in range(1, nd + 1)]
    s += [f"qr{i}_{j}" for i in range(1, ncu + 1) for j in range(1, nd + 1)]
    s += [f"mu{i}" for i in range(1, nparam + 1)]
    s += [f"n{k}" for k in range(1, nd + 1)]
    return tuple(s)


@dataclass
class OdeSpec:
    alpha: float = 1.0
    beta: float = 0.0
    sw: list = field(default_factory=list)


@dataclass
class BoundaryCondition:
    type: str
    data: list = field(default_factory=list)


@dataclass
class NumericalFluxSpec:
    trace: str = "switch"
    grad_trace: str = "opposite"
    tau: float = 1.0
    tau_over_h: bool | None = None
    uhat: list | None = None
    fhat: list | None = None


@dataclass
class PdeModel:
    kind: str
    ncu: int
    nd: int
    nw: int = 0
    nparam: int = 0
    mass: list = field(default_factory=list)
    flux: list = field(default_factory=list)
    source: list = field(default_factory=list)
    ode: OdeSpec | None = None
    numflux: NumericalFluxSpec = field(default_factory=NumericalFluxSpec)
    bcs: dict = field(default_factory=dict)
    init: dict = field(default_factory=dict)
    mu: np.ndarray = field(default_factory=lambda: np.zeros(0))
    tf: float = 0.0
    wavespeed: str | None = None

    def __post_init__(self):
        self.mu = np.asarray(self.mu, dtype=float)
        self._plans = {}

    @property
    def symbols(self):
        return reserved_symbols(self.ncu, self.nd, self.nw, self.nparam)

    def mu_bindings(self):
        return {f"mu{i + 1}": float(v) for i, v in enumerate(self.mu)}

    def _plan(self, key, texts, symbols=None):
        if key not in self._plans:
            self._plans[key] = compile_texts(list(texts), symbols or self.symbols)
        return self._plans[key]

    def flux_plan(self):
        return self._plan("flux", self.flux)

    def source_plan(self):
        return self._plan("source", self.source)

    def mass_plan(self):
        return self._plan("mass", self.mass)

    def sw_plan(self):
        return self._plan("sw", self.ode.sw)

    def wavespeed_plan(self):
        return None if self.wavespeed is None else \
            self._plan("wavespeed", [self.wavespeed])

    def bc_plan(self, tag):
        return self._plan(f"bc{tag}", self.bcs[tag].data)

    def init_exprs(self):
        keys = [f"u{i}" for i in range(1, self.ncu + 1)]
        if self.kind == "W":
            keys += [f"q{i}_{j}" for i in range(1, self.ncu + 1)
                     for j in range(1, self.nd + 1)]
        keys += [f"w{i}" for i in range(1, self.nw + 1)]
        return [self.init.get(k, "0") for k in keys]

    def init_plan(self):
        return self._plan("init", self.init_exprs())

    def uhat_plan(self):
        return None if self.numflux.uhat is None else self._plan(
            "uhat", self.numflux.uhat, face_symbols(self.ncu, self.nd, self.nparam))

    def fhat_plan(self):
        return None if self.numflux.fhat is None else self._plan(
            "fhat", self.numflux.fhat, face_symbols(self.ncu, self.nd, self.nparam))

    def is_steady(self):
        try:
            p = self.mass_plan()
        except ExprSyntaxError:
            return False
        return all(p.instructions[r] == ("const", 0.0) for r in p.outputs)


def validate(model):
    """Subset of the reference invariants (model.py:226-301); returns a list
    of message strings."""
    out = []
    if model.kind not in KINDS:
        return [f"kind must be one of {KINDS}, got {model.kind!r}"]
    if not (1 <= model.nd <= 3):
        out.append(f"nd must be 1..3, got {model.nd}")
    if model.ncu < 1:
        out.append(f"ncu must be >= 1, got {model.ncu}")
    if len(model.mass) != model.ncu:
        out.append(f"mass has {len(model.mass)} entries, expected ncu={model.ncu}")
    if len(model.flux) != model.ncu * model.nd:
        out.append(f"flux has {len(model.flux)} entries, expected "
                   f"ncu*nd={model.ncu * model.nd}")
    if len(model.source) != model.ncu:
        out.append(f"source has {len(model.source)} entries, expected "
                   f"ncu={model.ncu}")
    if len(model.mu) != model.nparam:
        out.append(f"mu has {len(model.mu)} values, expected "
                   f"nparam={model.nparam}")
    texts = list(model.mass) + list(model.flux) + list(model.source)
    for tag, bc in model.bcs.items():
        if bc.type not in BC_TYPES:
            out.append(f"bc tag {tag}: unknown type {bc.type!r}")
        if bc.type in ("dirichlet", "neumann") and len(bc.data) != model.ncu:
            out.append(f"bc tag {tag}: {len(bc.data)} data entries, expected "
                       f"ncu={model.ncu}")
        texts += list(bc.data)
    texts += list(model.init.values())
    if model.wavespeed is not None:
        texts.append(model.wavespeed)
    for t in texts:
        try:
            parse_expression(t, model.symbols)
        except ExprSyntaxError as e:
            out.append(str(e))
    return out


# ---------------------------------------------------------------------------
# builtin library (model.py:567-752)
# ---------------------------------------------------------------------------


def _nd(name, nd, allowed):
    nd = allowed[0] if nd is None else nd
    if nd not in allowed:
        raise ModelError(f"{name}: nd must be in {allowed}, got {nd}")
    return nd


def _poisson(nd):
    nd = _nd("poisson", nd, (1, 2, 3))
    return PdeModel(kind="D", ncu=1, nd=nd, mass=["0"],
                    flux=[f"q1_{j + 1}" for j in range(nd)], source=["0"],
                    init={"u1": "0"})


def _convection_diffusion(nd):
    nd = _nd("convection_diffusion", nd, (1, 2, 3))
    flux = [f"mu{j + 1}*u1 + mu{nd + 1}*q1_{j + 1}" for j in range(nd)]
    speed = "abs(" + "+".join(f"mu{j + 1}*n{j + 1}" for j in range(nd)) + ")"
    return PdeModel(kind="D", ncu=1, nd=nd, nparam=nd + 1, mass=["1"],
                    flux=flux, source=["0"], mu=np.ones(nd + 1),
                    wavespeed=speed, init={"u1": "0"})


def _linear_convection(nd):
    nd = _nd("linear_convection", nd, (1, 2, 3))
    speed = "abs(" + "+".join(f"mu{j + 1}*n{j + 1}" for j in range(nd)) + ")"
    return PdeModel(kind="C", ncu=1, nd=nd, nparam=nd, mass=["1"],
                    flux=[f"mu{j + 1}*u1" for j in range(nd)], source=["0"],
                    mu=np.ones(nd), wavespeed=speed, init={"u1": "0"})


def _burgers(nd):
    nd = _nd("burgers", nd, (1, 2))
    speed = "abs(u1*(" + "+".join(f"n{j + 1}" for j in range(nd)) + "))"
    return PdeModel(kind="C", ncu=1, nd=nd, mass=["1"], flux=["u1*u1/2"] * nd,
                    source=["0"], wavespeed=speed, init={"u1": "0"})


def _euler(nd):
    nd = _nd("euler", nd, (2, 3))
    ncu = nd + 2
    e = ncu
    ke = "+".join(f"u{k}*u{k}" for k in range(2, nd + 2))
    p = f"(mu1-1)*(u{e} - (({ke})/u1)/2)"
    flux = []
    for i in range(1, ncu + 1):
        for j in range(1, nd + 1):
            vj = f"u{j + 1}/u1"
            if i == 1:
                flux.append(f"u{j + 1}")
            elif i == e:
                flux.append(f"(u{e} + {p})*{vj}")
            else:
                flux.append(f"u{i}*{vj}" + (f" + {p}" if i == j + 1 else ""))
    vn = "+".join(f"u{j + 1}/u1*n{j}" for j in range(1, nd + 1))
    init = {"u1": "1", f"u{e}": "2.5"}
    init.update({f"u{k}": "0" for k in range(2, nd + 2)})
    return PdeModel(kind="C", ncu=ncu, nd=nd, nparam=1, mass=["1"] * ncu,
                    flux=flux, source=["0"] * ncu, mu=np.array([1.4]),
                    wavespeed=f"abs({vn}) + sqrt(mu1*({p})/u1)", init=init)


def _linear_elasticity(nd):
    nd = _nd("linear_elasticity", nd, (2, 3))
    tr = "+".join(f"q{i}_{i}" for i in range(1, nd + 1))
    flux = []
    for i in range(1, nd + 1):
        for j in range(1, nd + 1):
            s = f"-(mu2*(q{i}_{j} + q{j}_{i}))"
            flux.append(s + (f" - mu1*({tr})" if i == j else ""))
    return PdeModel(kind="D", ncu=nd, nd=nd, nparam=2, mass=["0"] * nd,
                    flux=flux, source=["0"] * nd, mu=np.array([1.0, 1.0]),
                    init={f"u{i}": "0" for i in range(1, nd + 1)})


def _shallow_water(nd):
    _nd("shallow_water", nd, (2,))
    flux = ["u2", "u3", "u2*u2/u1 + mu1*u1*u1/2", "u2*u3/u1",
            "u2*u3/u1", "u3*u3/u1 + mu1*u1*u1/2"]
    return PdeModel(kind="C", ncu=3, nd=2, nparam=1, mass=["1"] * 3, flux=flux,
                    source=["0"] * 3, mu=np.array([1.0]),
                    wavespeed="abs(u2/u1*n1 + u3/u1*n2) + sqrt(mu1*u1)",
                    init={"u1": "1", "u2": "0", "u3": "0"})


def _compressible_ns(nd):
    """2D compressible Navier-Stokes, kind D (model.py:677-712 restated):
    gamma = mu1, viscosity = mu2, Prandtl = mu3; q_ij = -d(u_i)/dx_j."""
    _nd("compressible_ns", nd, (2,))
    ke = "u2*u2+u3*u3"
    p = f"(mu1-1)*(u4 - (({ke})/u1)/2)"
    vel = ("u2/u1", "u3/u1")

    def dv(i, j):            # d(velocity_i)/dx_j from the conserved gradients
        return f"(({vel[i]})*q1_{j + 1} - q{i + 2}_{j + 1})/u1"

    txx = f"mu2*(4*({dv(0, 0)})/3 - 2*({dv(1, 1)})/3)"
    tyy = f"mu2*(4*({dv(1, 1)})/3 - 2*({dv(0, 0)})/3)"
    txy = f"mu2*(({dv(0, 1)}) + ({dv(1, 0)}))"
    T = f"(u4 - ({ke})/(2*u1))/u1"

    def dT(j):
        return (f"((({T})*q1_{j} - q4_{j} + (({vel[0]})*q2_{j} + ({vel[1]})*q3_{j}) - "
                f"(({ke})/(2*u1))/u1*q1_{j})/u1)")

    k = "mu1*mu2/mu3"
    vx, vy = vel
    flux = ["u2", "u3",
            f"u2*({vx}) + {p} - ({txx})", f"u2*({vy}) - ({txy})",
            f"u3*({vx}) - ({txy})", f"u3*({vy}) + {p} - ({tyy})",
            f"(u4 + {p})*({vx}) - ({vx})*({txx}) - ({vy})*({txy}) - ({k})*({dT(1)})",
            f"(u4 + {p})*({vy}) - ({vx})*({txy}) - ({vy})*({tyy}) - ({k})*({dT(2)})"]
    return PdeModel(kind="D", ncu=4, nd=2, nparam=3, mass=["1"] * 4, flux=flux,
                    source=["0"] * 4, mu=np.array([1.4, 1e-3, 0.72]),
                    wavespeed=f"abs({vx}*n1 + {vy}*n2) + sqrt(mu1*({p})/u1)",
                    init={"u1": "1", "u2": "0", "u3": "0", "u4": "2.5"})


def _wave(nd):
    """Scalar wave equation, kind W (model.py:715-727 restated): du/dt +
    c^2 div(q) = 0, dq/dt + grad(u) = 0, displacement dw/dt = u; c = mu1."""
    nd = _nd("wave", nd, (1, 2, 3))
    init = {"u1": "0", "w1": "0"}
    init.update({f"q1_{j + 1}": "0" for j in range(nd)})
    return PdeModel(kind="W", ncu=1, nd=nd, nw=1, nparam=1, mass=["1"],
                    flux=[f"mu1*mu1*q1_{j + 1}" for j in range(nd)], source=["0"],
                    ode=OdeSpec(alpha=1.0, beta=0.0, sw=["u1"]), mu=np.array([1.0]),
                    wavespeed="mu1", init=init)


_BUILTINS = {
    "wave": _wave,
    "shallow_water": _shallow_water,
    "compressible_ns": _compressible_ns,
    "poisson": _poisson,
    "convection_diffusion": _convection_diffusion,
    "linear_convection": _linear_convection,
    "burgers": _burgers,
    "euler": _euler,
    "linear_elasticity": _linear_elasticity,
}


def builtin_model(name, nd=None, mu=None):
    if name not in _BUILTINS:
        raise ModelError(f"unknown builtin model {name!r}")
    m = _BUILTINS[name](nd)
    if mu is not None:
        mu = np.asarray(mu, dtype=float)
        if len(mu) != m.nparam:
            raise ModelError(f"{name}: expected {m.nparam} parameters, got "
                             f"{len(mu)}")
        m.mu = mu
    d = validate(m)
    if d:
        raise ModelError(f"builtin {name} failed validation: " + "; ".join(d))
    return m


# ---------------------------------------------------------------------------
# model files (grammar of model.py:317-332)
# ---------------------------------------------------------------------------


def parse_model_text(text):
    sections = []
    cur = None
    for ln, raw in enumerate(text.splitlines(), start=1):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        if line.startswith("["):
            if "]" not in line:
                raise ModelFileError("unterminated section header", ln)
            head, rest = line[1:].split("]", 1)
            parts = head.split()
            if not parts:
                raise ModelFileError("empty section header", ln)
            attrs = {}
            for item in parts[1:] + rest.split():
                if "=" not in item:
                    raise ModelFileError(f"bad header item {item!r}", ln)
                k, v = item.split("=", 1)
                attrs[k.strip()] = v.strip()
            cur = [parts[0], attrs, [], ln]
            sections.append(cur)
            continue
        if cur is None:
            raise ModelFileError("assignment before any section", ln)
        if "=" not in line:
            raise ModelFileError(f"expected key=value, got {line!r}", ln)
        k, v = line.split("=", 1)
        cur[2].append((k.strip(), v.strip()))

    named, bcs_raw = {}, []
    for name, attrs, items, ln in sections:
        if name == "bc":
            bcs_raw.append((attrs, items, ln))
            continue
        if name in named:
            raise ModelFileError(f"duplicate section [{name}]", ln)
        if name != "model":
            items = list(attrs.items()) + items
            attrs = {}
        named[name] = (attrs, dict(items), ln)
    if "model" not in named:
        raise ModelFileError("missing [model] section")
    attrs, body, ln = named["model"]
    for k, v in body.items():
        attrs.setdefault(k, v)
    try:
        kind = attrs["kind"]
        ncu, nd = int(attrs["ncu"]), int(attrs["nd"])
        nw = int(attrs.get("nw", "0"))
        nparam = int(attrs.get("nparam", "0"))
        tf = float(attrs.get("tf", "0.0"))
    except KeyError as e:
        raise ModelFileError(f"[model] missing attribute {e}", ln) from None
    except ValueError as e:
        raise ModelFileError(f"[model]: {e}", ln) from None

    def ordered(sec, keys, default):
        if sec not in named:
            return [default] * len(keys)
        _, vals, sln = named[sec]
        miss = [k for k in keys if k not in vals]
        if miss:
            raise ModelFileError(f"[{sec}] missing entry {miss[0]}", sln)
        extra = set(vals) - set(keys)
        if extra:
            raise ModelFileError(f"[{sec}] unexpected entries {sorted(extra)}", sln)
        return [vals[k] for k in keys]

    mass = ordered("mass", [f"m{i}" for i in range(1, ncu + 1)], "1")
    flux = ordered("flux", [f"f{i}_{j}" for i in range(1, ncu + 1)
                            for j in range(1, nd + 1)], "0")
    source = ordered("source", [f"s{i}" for i in range(1, ncu + 1)], "0")
    mu = np.zeros(nparam)
    if "mu" in named:
        for k, v in named["mu"][1].items():
            if not (k.startswith("mu") and k[2:].isdigit()) or \
                    not (1 <= int(k[2:]) <= nparam):
                raise ModelFileError(f"[mu] bad key {k!r}", named["mu"][2])
            mu[int(k[2:]) - 1] = float(v)
    ode = None
    if "ode" in named:
        vals = named["ode"][1]
        sw = []
        for i in range(1, nw + 1):
            if f"sw{i}" not in vals:
                raise ModelFileError(f"[ode] missing sw{i}", named["ode"][2])
            sw.append(vals[f"sw{i}"])
        ode = OdeSpec(alpha=float(vals.get("alpha", "1")),
                      beta=float(vals.get("beta", "0")), sw=sw)
    numflux, wavespeed = NumericalFluxSpec(), None
    if "numflux" in named:
        vals = named["numflux"][1]
        oh = vals.get("tau_over_h")
        numflux = NumericalFluxSpec(
            trace=vals.get("trace", "switch"),
            grad_trace=vals.get("grad_trace", "opposite"),
            tau=float(vals.get("tau", "1")),
            tau_over_h=None if oh is None else bool(int(oh)))
        wavespeed = vals.get("wavespeed")
        uh = [vals[k] for k in sorted(vals) if k.startswith("uhat")]
        fh = [vals[k] for k in sorted(vals) if k.startswith("fhat")]
        numflux.uhat = uh or None
        numflux.fhat = fh or None
    bcs = {}
    for a, items, sln in bcs_raw:
        try:
            tag, btype = int(a["tag"]), a["type"]
        except KeyError as e:
            raise ModelFileError(f"[bc] missing attribute {e}", sln) from None
        data = dict(items)
        bcs[tag] = BoundaryCondition(
            type=btype,
            data=[data[f"g{i}"] for i in range(1, ncu + 1) if f"g{i}" in data])
    init = dict(named["init"][1]) if "init" in named else {}
    return PdeModel(kind=kind, ncu=ncu, nd=nd, nw=nw, nparam=nparam, mass=mass,
                    flux=flux, source=source, ode=ode, numflux=numflux, bcs=bcs,
                    init=init, mu=mu, tf=tf, wavespeed=wavespeed)


def load_model(path):
    with open(path) as f:
        m = parse_model_text(f.read())
    d = validate(m)
    if d:
        raise ModelError("model validation failed:\n" + "\n".join(d))
    return m
