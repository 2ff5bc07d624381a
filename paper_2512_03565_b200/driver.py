"""Force-phase entry points (the drop-in seam, driver.py:107-129).

``force_phase`` keeps the reference's signature and semantics: it builds the
configured container around the owned particles, derives the periodic
images, runs one force computation and OVERWRITES ``owned.force_*`` with the
total forces, returning the KernelStats.  Buffers may live on the host
(numpy SoA with the reference's field names, e.g. a reference
``ParticleBuffer``) or on the device (our ``ParticleBuffer`` on CUDA); host
buffers are copied to HBM and the forces copied back inside the call.
"""

from __future__ import annotations

from .containers import LinkedCellsContainer, device_soa
from .domain import as_box
from .errors import ConfigurationError
from .kernels import KernelStats, as_pattern, validate_vector_width
from .tuning import Configuration, ContainerKind


def make_container(kind, box, params, cluster_size=None, rebuild_period=None, device=None):
    kind = ContainerKind(getattr(kind, "value", kind))
    kw = {} if rebuild_period is None else {"rebuild_period": rebuild_period}
    if kind is ContainerKind.LINKED_CELLS:
        return LinkedCellsContainer(box, params, device=device, **kw)
    if kind is ContainerKind.VERLET_LISTS:
        from .verlet_lists import VerletListContainer
        return VerletListContainer(box, params, device=device, **kw)
    from .clusters import VerletClusterContainer
    if cluster_size is None:
        raise ConfigurationError("cluster container needs a cluster size")
    return VerletClusterContainer(box, params, cluster_size, device=device, **kw)


def force_phase(owned, box, params, config: Configuration, vector_width: int,
                cluster_size: int | None = None, energy: bool = False) -> KernelStats:
    """One standalone force computation through the device container pipeline."""
    validate_vector_width(vector_width)
    if not isinstance(config, Configuration):
        config = Configuration(config.container, config.traversal, config.newton3,
                               config.pattern)
    if not config.is_valid():
        raise ConfigurationError(f"invalid configuration {config.label!r}")
    box = as_box(box)
    dev_owned = device_soa(owned)
    cont = make_container(config.container, box, params,
                          cluster_size=config.cluster_size or cluster_size or vector_width)
    lean = _one_shot(cont)
    cont.rebuild(dev_owned)
    if not lean:           # (a lean rebuild has loaded the current positions)
        cont.refresh(dev_owned)
    stats = _compute_once(cont, config, vector_width, energy)
    cont.collect_forces(dev_owned)
    if dev_owned is not owned:
        _write_forces_back(owned, dev_owned)
    return stats


def _one_shot(cont) -> bool:
    """Mark a container as built for one force computation; True when its
    rebuild then loads the current positions itself (Verlet lists: no pos4 /
    SoA copies, no snapshots of the build-time state, plain list order if
    lists are needed at all)."""
    if hasattr(cont, "bank_rounds"):
        # the bank-aware list order pays for its pass only when lists are reused
        cont.bank_rounds = -1
    if hasattr(cont, "one_shot"):
        cont.one_shot = True
        return bool(cont.segmented)
    return False


def _compute_once(cont, config, vector_width: int, energy: bool) -> KernelStats:
    """The force computation of a container built for this one call: where
    the container has a list-free kernel for it (Verlet lists, N x 1) that one
    runs, else the regular ``compute_forces``."""
    once = getattr(cont, "compute_forces_once", None)
    stats = None
    if once is not None:
        stats = once(config.traversal, config.newton3, as_pattern(config.pattern),
                     vector_width, energy=energy)
    if stats is None:
        stats = cont.compute_forces(config.traversal, config.newton3,
                                    as_pattern(config.pattern), vector_width, energy=energy)
    return stats


def force_phase_bricks(owned, dec, params, config: Configuration, vector_width: int,
                        cluster_size: int | None = None, energy: bool = False) -> KernelStats:
    """``force_phase`` for one brick of a domain decomposition (one rank per
    GPU): ``owned`` holds this rank's particles (host or device SoA buffer,
    positions inside the brick), ``dec`` the BrickDecomposition.  The ghost
    layer (interaction length thick, periodic images across the global box
    included) is planned and exchanged with the neighbouring ranks inside
    the call, the container is built over [owned | ghosts], one force
    computation runs and ``owned.force_*`` is overwritten.  The returned
    statistics are this rank's (owned-ghost pairs counted on the owned side,
    traversals.py:157-160); sum them over ranks for the global figures."""
    import torch

    from .particles import ParticleBuffer
    validate_vector_width(vector_width)
    if not config.is_valid():
        raise ConfigurationError(f"invalid configuration {config.label!r}")
    dev_owned = device_soa(owned)
    pos = torch.stack([dev_owned.pos_x, dev_owned.pos_y, dev_owned.pos_z], dim=1)
    ghost_rows = dec.plan(pos)
    ghosts = ParticleBuffer.empty(ghost_rows.shape[0], device=pos.device)
    ghosts.pos_x.copy_(ghost_rows[:, 0])
    ghosts.pos_y.copy_(ghost_rows[:, 1])
    ghosts.pos_z.copy_(ghost_rows[:, 2])
    cont = make_container(config.container, dec.local_box(), params,
                          cluster_size=config.cluster_size or cluster_size or vector_width)
    lean = _one_shot(cont)
    cont.rebuild(dev_owned, ghosts)
    if not lean:
        cont.refresh(dev_owned, ghosts)
    stats = _compute_once(cont, config, vector_width, energy)
    cont.collect_forces(dev_owned)
    if dev_owned is not owned:
        _write_forces_back(owned, dev_owned)
    return stats


def _write_forces_back(host, dev) -> None:
    import torch
    for name in ("force_x", "force_y", "force_z"):
        dst = getattr(host, name)
        val = getattr(dev, name)
        if isinstance(dst, torch.Tensor):
            dst.copy_(val)   # direct device -> (pinned) host DMA
        else:
            torch.from_numpy(dst).copy_(val)
